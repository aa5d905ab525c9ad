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
           "ExtrapolationResult", "ReconstructionCoefficients", "QrFactorization",
           "build_difference_matrix", "mgs_qr", "small_svd", "gamma_mpe", "gamma_rre",
           "gamma_svdmpe", "reconstruction_coefficients", "reconstruct", "extrapolate_once",
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


@dataclass(frozen=True)
class QrFactorization:
    """Thin QR of the difference matrix (extrapolation.py:97-109).  ``Q`` is
    an [N, kappa+1] CUDA tensor (a column-major view), ``R`` a host array."""

    Q: object
    R: np.ndarray
    effective_rank: int
    rank_tolerance: float


# --------------------------------------------------------------------- factor-level API
# The pieces extrapolate_once chains together, for callers that use them on
# their own (extrapolation.py:154-316).  The N-length vector work (differences,
# Gram-Schmidt projections, reconstruction) runs in libredve_b200's vector
# primitives; the (kappa+1)^2 triangular algebra is host arithmetic, as in the
# reference.


def _dev_rows(v):
    t, _ = _io.to_device(v)
    return t.reshape(t.shape[0], -1).contiguous()


def _dot(x, y):
    out = C.c_double()
    ctx = nat.context()
    nat.check(nat.library().redve_vec_dot(ctx, x.numel(), nat.dptr(x), nat.dptr(y), C.byref(out)),
              ctx)
    return out.value


def _axpby(a, x, b, y):
    ctx = nat.context()
    nat.check(nat.library().redve_vec_axpby(ctx, y.numel(), float(a), nat.dptr(x), float(b),
                                            nat.dptr(y)), ctx)


def build_difference_matrix(window: VectorSequenceWindow):
    """N x (kappa+1) matrix whose column i is x_{m+i+1} - x_{m+i}
    (extrapolation.py:154-156); a column-major view of a device buffer."""
    rows = _dev_rows(window.vectors)
    diff = rows[1:].clone()
    for i in range(diff.shape[0]):
        _axpby(-1.0, rows[i], 1.0, diff[i])
    return diff.T


def mgs_qr(u, rank_tolerance: float = 1e-12) -> QrFactorization:
    """Modified Gram-Schmidt with two projection sweeps per column and the
    relative rank cut r_ii < tol * r_11 (extrapolation.py:159-196)."""
    if rank_tolerance <= 0:
        raise ValueError("rank_tolerance must be positive")
    t, _ = _io.to_device(u)
    if t.dim() != 2:
        raise ValueError("mgs_qr expects an N x k matrix")
    cols = t.T.contiguous()  # column i contiguous
    k = cols.shape[0]
    q = _io.torch_mod().zeros_like(cols)
    r = np.zeros((k, k))
    r11 = 0.0
    effective = k
    for i in range(k):
        v = cols[i].clone()
        for _sweep in range(2):
            for j in range(i):
                proj = _dot(q[j], v)
                r[j, i] += proj
                _axpby(-proj, q[j], 1.0, v)
        rii = float(np.sqrt(_dot(v, v)))
        r[i, i] = rii
        if i == 0:
            if rii < 1e-300:
                raise ZeroFirstColumn("first difference column is zero")
            r11 = rii
        elif rii < rank_tolerance * r11:
            effective = i
            break
        _axpby(0.0, v, 1.0 / rii, v)
        q[i].copy_(v)
    return QrFactorization(Q=q.T, R=r, effective_rank=effective, rank_tolerance=rank_tolerance)


def small_svd(r):
    """SVD of the small triangular factor (extrapolation.py:199-214)."""
    r = np.asarray(r, dtype=np.float64)
    if r.ndim != 2 or r.shape[0] != r.shape[1]:
        raise ValueError("small_svd expects a square matrix")
    if r.shape[0] > 64:
        raise ValueError("small_svd is intended for windows of order <= 63")
    try:
        return np.linalg.svd(r)
    except np.linalg.LinAlgError as exc:  # pragma: no cover - pathological input
        raise NoConvergence(str(exc)) from exc


def _require_full_rank(qr: QrFactorization) -> int:
    ncols = qr.R.shape[0]
    if qr.effective_rank != ncols:
        raise RankDeficient(f"effective rank {qr.effective_rank} < {ncols}; shrink the window order")
    return ncols - 1


def _normalized(method, c, denom):
    gamma = c / denom
    return ExtrapolationWeights(method=method, c=c, gamma=gamma,
                                stability_sum=float(np.abs(gamma).sum()))


def _upper_solve(r, b, trans=False):
    from scipy.linalg import solve_triangular

    return solve_triangular(r, b, trans="T" if trans else "N", lower=False)


def gamma_mpe(qr: QrFactorization) -> ExtrapolationWeights:
    """MPE weights; DegenerateSum when sum(c) vanishes (extrapolation.py:241-260)."""
    kappa = _require_full_rank(qr)
    cp = _upper_solve(qr.R[:kappa, :kappa], -qr.R[:kappa, kappa])
    c = np.append(cp, 1.0)
    s = float(c.sum())
    if abs(s) < 1e-12 * float(np.abs(c).sum()) or not np.isfinite(s):
        raise DegenerateSum("MPE coefficient sum vanished")
    return _normalized(MPE, c, s)


def gamma_rre(qr: QrFactorization) -> ExtrapolationWeights:
    """RRE weights from (R^T R) d = 1 (extrapolation.py:263-273)."""
    _require_full_rank(qr)
    d = _upper_solve(qr.R, _upper_solve(qr.R, np.ones(qr.R.shape[0]), trans=True))
    return _normalized(RRE, d, float(d.sum()))


def gamma_svdmpe(qr: QrFactorization) -> ExtrapolationWeights:
    """SVD-MPE weights: right singular vector of the smallest singular value
    (extrapolation.py:276-284)."""
    _require_full_rank(qr)
    _, _, vt = small_svd(qr.R)
    v = vt[-1].copy()
    s = float(v.sum())
    if abs(s) < 1e-12 or not np.isfinite(s):
        raise DegenerateSum("SVD-MPE singular-vector sum vanished")
    return _normalized(SVDMPE, v, s)


def reconstruction_coefficients(gamma, r) -> ReconstructionCoefficients:
    """xi_j = 1 - (gamma_0 + ... + gamma_j), eta = R xi (extrapolation.py:295-305)."""
    gamma = np.asarray(gamma, dtype=np.float64)
    kappa = len(gamma) - 1
    xi = 1.0 - np.cumsum(gamma[:kappa])
    eta = np.asarray(r)[:kappa, :kappa] @ xi
    return ReconstructionCoefficients(xi=xi, eta=eta)


def reconstruct(window: VectorSequenceWindow, qr: QrFactorization, w: ExtrapolationWeights):
    """x_m + Q (R xi) through the factors (extrapolation.py:308-316); a device
    tensor when the window lives on the device, else a numpy array."""
    kappa = window.kappa
    if len(w.gamma) != kappa + 1:
        raise ValueError(f"{len(w.gamma)} weights for a window of order {kappa}")
    coeffs = reconstruction_coefficients(w.gamma, qr.R)
    rows = _dev_rows(window.vectors)
    out = rows[0].clone()
    qcols = qr.Q.T if _io.is_tensor(qr.Q) else _dev_rows(np.asarray(qr.Q).T)
    for j in range(kappa):
        _axpby(float(coeffs.eta[j]), qcols[j].contiguous(), 1.0, out)
    out = out.reshape(window.vectors.shape[1:])
    return out if _io.is_tensor(window.vectors) else out.cpu().numpy()


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
