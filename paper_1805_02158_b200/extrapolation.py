"""Vector extrapolation (MPE / RRE / SVD-MPE) -- drop-in for ``redve.extrapolation``.

``extrapolate_once`` runs in libredve_b200: one fp64 Gram pass over the
window's differences (deterministic reduction), the (kappa+1)^2 decision
logic on the device, the exact modified-Gram-Schmidt route when the Gram
route cannot resolve the rank question, and the recombination kernel.  The
result types and fallback policy are the reference's
(extrapolation.py:62-146, 319-386).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _io
from . import _native as nat
from .errors import DegenerateSum, NoConvergence, RankDeficient, ZeroFirstColumn

MPE = "mpe"
RRE = "rre"
SVDMPE = "svdmpe"
METHODS = (MPE, RRE, SVDMPE)

__all__ = ["MPE", "RRE", "SVDMPE", "METHODS", "VectorSequenceWindow", "ExtrapolationWeights",
           "ExtrapolationResult", "ReconstructionCoefficients", "extrapolate_once",
           "extrapolate_batch", "ZeroFirstColumn", "DegenerateSum", "RankDeficient",
           "NoConvergence"]


@dataclass(frozen=True)
class VectorSequenceWindow:
    """kappa+2 consecutive iterates as rows (extrapolation.py:62-93).

    ``vectors`` may be a numpy array or a CUDA tensor (kept on the device)."""

    vectors: object
    m: int = 0

    def __post_init__(self):
        v = self.vectors
        if _io.is_tensor(v):
            torch = _io.torch_mod()
            v = v.to(dtype=torch.float64)
            if v.dim() != 2 or v.shape[0] < 3:
                raise ValueError("window needs at least kappa+2 = 3 equal-length vectors")
            if not bool(torch.isfinite(v).all()):
                raise ValueError("window contains non-finite entries")
        else:
            v = np.asarray(v, dtype=np.float64)
            if v.ndim != 2 or v.shape[0] < 3:
                raise ValueError("window needs at least kappa+2 = 3 equal-length vectors")
            if not np.all(np.isfinite(v)):
                raise ValueError("window contains non-finite entries")
        if self.m < 0:
            raise ValueError("m must be nonnegative")
        object.__setattr__(self, "vectors", v)

    @classmethod
    def from_iterates(cls, iterates, m: int = 0) -> "VectorSequenceWindow":
        return cls(np.array([np.asarray(x, dtype=np.float64).ravel() for x in iterates]), m=m)

    @property
    def kappa(self) -> int:
        return self.vectors.shape[0] - 2

    @property
    def dimension(self) -> int:
        return self.vectors.shape[1]


@dataclass(frozen=True)
class ExtrapolationWeights:
    """Raw coefficients c and normalised weights gamma (extrapolation.py:111-124)."""

    method: str
    c: np.ndarray
    gamma: np.ndarray
    stability_sum: float
    fallback_from: str | None = None


class ReconstructionCoefficients(NamedTuple):
    xi: np.ndarray
    eta: np.ndarray


@dataclass(frozen=True)
class ExtrapolationResult:
    """Outcome of one extrapolation attempt (extrapolation.py:132-146)."""

    vector: object
    weights: ExtrapolationWeights | None
    converged: bool
    extrapolated: bool
    kappa_used: int


def _weights_from(res: "nat.VeResultC", requested: str):
    if not res.extrapolated and not (res.kappa_used > 0):
        return None
    k = res.kappa_used
    gamma = np.array(res.gamma[: k + 1])
    c = np.array(res.c[: k + 1])
    used = nat.VE_NAMES[res.method]
    return ExtrapolationWeights(
        method=used, c=c, gamma=gamma, stability_sum=float(res.stability_sum),
        fallback_from=requested if res.fallback else None)


def extrapolate_batch(windows, method: str = MPE, rank_tolerance: float = 1e-12):
    """B windows at once: ``windows`` is [B, kappa+2, n] (numpy or CUDA tensor).
    Returns (vectors [B, n], list of per-window result dicts)."""
    if method not in METHODS:
        raise ValueError(f"method must be one of {METHODS}, got {method!r}")
    t, from_np = _io.to_device(windows)
    if t.dim() != 3 or t.shape[1] < 3:
        raise ValueError("windows must be [B, kappa+2 >= 3, n]")
    B, rows, n = t.shape
    out = _io.empty((B, n))
    res = (nat.VeResultC * B)()
    ctx = nat.context()
    nat.check(nat.library().redve_extrapolate(ctx, B, rows, n, nat.dptr(t), nat.VE_CODES[method],
                                              float(rank_tolerance), nat.dptr(out), res), ctx)
    return _io.to_host(out, from_np), list(res)


def extrapolate_once(window: VectorSequenceWindow, method: str = MPE,
                     rank_tolerance: float = 1e-12) -> ExtrapolationResult:
    """Differences -> Gram/QR -> weights -> reconstruction, with the reference's
    fallback policy (extrapolation.py:319-386)."""
    if method not in METHODS:
        raise ValueError(f"method must be one of {METHODS}, got {method!r}")
    if rank_tolerance <= 0:
        raise ValueError("rank_tolerance must be positive")
    v = window.vectors
    vecs, res = extrapolate_batch(v[None] if not _io.is_tensor(v) else v.unsqueeze(0), method,
                                  rank_tolerance)
    r = res[0]
    vec = vecs[0]
    if r.converged:
        return ExtrapolationResult(vec, None, True, False, 0)
    if not r.extrapolated:
        return ExtrapolationResult(vec, None, False, False, 0)
    return ExtrapolationResult(vec, _weights_from(r, method), False, True, int(r.kappa_used))
