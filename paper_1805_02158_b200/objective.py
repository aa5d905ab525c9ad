"""Denoiser-regularised objective and its fixed-point step -- drop-in for ``redve.objective``.

E(x) = ||H x - y||^2/(2 sigma^2) + alpha/2 x.(x - f(x)); the fixed-point step
(H^T H/sigma^2 + alpha I)^{-1}(H^T y/sigma^2 + alpha f(x)) runs in libredve_b200
(objective.py:44-135): Fourier route for circulant H with the denoiser fused
into the first FFT pass.
"""

from __future__ import annotations

import numpy as np

from . import _io
from .batch import RedBatch
from .errors import CgNoConvergence
from .imaging import as_image
from .solvers import FixedPointProblem

CG_RTOL = 1e-6
CG_MAXITER = 200
CG_ABORT_RESIDUAL = 1e-4

__all__ = ["RedObjective", "as_fixed_point_problem", "default_step_size",
           "check_local_homogeneity", "check_passivity", "CgNoConvergence"]


class RedObjective:
    """objective.py:44-121 -- same constructor and methods, device arithmetic."""

    def __init__(self, forward, y, sigma: float, alpha: float, denoiser):
        if sigma <= 0:
            raise ValueError("sigma must be > 0")
        if alpha <= 0:
            raise ValueError("alpha must be > 0")
        y = as_image(y)
        if y.shape != tuple(forward.out_shape):
            raise ValueError(f"y shape {y.shape} != operator output {forward.out_shape}")
        self.forward = forward
        self.y = y
        self.sigma = float(sigma)
        self.alpha = float(alpha)
        self.denoiser = denoiser
        self._batch = RedBatch(forward, y, sigma, alpha, denoiser)
        self._ref_batch = None  # (reference array, RedBatch with that reference)

    @property
    def device_solvable(self) -> bool:
        return self._batch.device_solvable

    # -- objective pieces ------------------------------------------------------
    def _terms(self, x):
        cost, fid, reg, _ = self._batch.cost_terms(np.asarray(x, dtype=np.float64))
        return float(cost[0]), float(fid[0]), float(reg[0])

    def data_fidelity(self, x) -> float:
        return self._terms(x)[1]

    def regularizer(self, x) -> float:
        return self._terms(x)[2]

    def cost(self, x) -> float:
        return self._terms(x)[0]

    def gradient(self, x):
        """H^T (H x - y)/sigma^2 + alpha (x - f(x))  (objective.py:90-93)."""
        out, from_np = self._batch.gradient(x)
        return _io.to_host(out[0], from_np)

    def fp_step(self, x):
        out, from_np = self._batch.fp_step(x)
        return _io.to_host(out[0], from_np)

    # -- device solve used by solvers.solve ------------------------------------
    def _device_solve(self, x0, config, method, reference):
        # PSNR is recorded against exactly this solve's reference (None: no PSNR)
        batch = self._batch
        if reference is not None:
            ref = np.asarray(reference, dtype=np.float64).reshape(self.forward.in_shape)
            held = self._ref_batch
            if held is None or held[0].shape != ref.shape or not np.array_equal(held[0], ref):
                held = (ref.copy(), RedBatch(self.forward, self.y, self.sigma, self.alpha,
                                             self.denoiser, ref))
                self._ref_batch = held
            batch = held[1]
        x0 = np.asarray(x0, dtype=np.float64).reshape(self.forward.in_shape)
        if x0.size != int(np.prod(self.forward.in_shape)):
            raise ValueError("x0 has the wrong dimension")
        res = batch.solve(x0, config, method)
        res.raise_for(0)
        return res.x[0].reshape(-1).cpu().numpy(), res.trace(0)


def as_fixed_point_problem(obj: RedObjective, reference=None) -> FixedPointProblem:
    """objective.py:124-135 -- flat-vector adapter; ``red`` routes solve() to the device."""
    shape = tuple(obj.forward.in_shape)
    n = shape[0] * shape[1]
    ref = None if reference is None else np.asarray(reference, dtype=np.float64).ravel()
    return FixedPointProblem(
        dimension=n,
        step=lambda v: np.asarray(obj.fp_step(np.asarray(v).reshape(shape))).ravel(),
        objective=lambda v: obj.cost(np.asarray(v).reshape(shape)),
        gradient=lambda v: np.asarray(obj.gradient(np.asarray(v).reshape(shape))).ravel(),
        reference=ref,
        red=obj,
    )


def default_step_size(sigma: float, alpha: float) -> float:
    """objective.py:138-145."""
    return sigma**2 / (1.0 + 2.0 * alpha * sigma**2)


def check_local_homogeneity(denoiser, x, c: float) -> float:
    """objective.py:153-158."""
    x = as_image(x)
    fx = np.asarray(denoiser(x))
    dev = np.linalg.norm(np.asarray(denoiser(c * x)) - c * fx)
    return float(dev / (np.linalg.norm(fx) + 1e-12))


def check_passivity(denoiser, x, iterations: int = 20, seed: int = 0) -> float:
    """objective.py:161-184 (power iteration on finite-difference JVPs)."""
    x = as_image(x)
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(x.shape)
    v /= np.linalg.norm(v)
    fx = np.asarray(denoiser(x))
    scale = max(float(np.linalg.norm(x)), 1.0)
    estimate = 0.0
    for _ in range(iterations):
        h = 1e-4 * scale
        jv = (np.asarray(denoiser(x + h * v)) - fx) / h
        estimate = float(np.linalg.norm(jv))
        if estimate == 0.0:
            return 0.0
        v = jv / estimate
    return estimate
