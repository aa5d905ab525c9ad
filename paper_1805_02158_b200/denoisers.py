"""Denoiser plug-ins f(x) -- drop-in for ``redve.denoisers``.

Each built-in carries a native descriptor so ``RedObjective`` can fuse it into
the device fixed-point step; calling it directly runs the same CUDA stencil
on one image or a batch.  Any other callable ``f(x: ndarray[H, W]) -> ndarray``
still works with ``RedObjective`` (the reference's callable-denoiser
protocol, denoisers.py:1-8); it is then evaluated by the caller's code.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _io
from . import _native as nat
from .imaging import Psf, make_psf

__all__ = ["Identity", "GaussianFilter", "Median3", "NotLinear", "materialize_dense",
           "BUILTIN_DENOISERS", "denoise"]


class NotLinear(TypeError):
    """Dense matrix requested for a nonlinear denoiser (denoisers.py:17-18)."""


class _Native:
    kind = nat.DN_IDENTITY
    linear = True

    def _desc(self):
        d = nat.DenoiserDesc()
        d.kind = self.kind
        self._fill(d)
        return d

    def _fill(self, d):
        pass

    def __call__(self, x):
        t, from_np = _io.to_device(x)
        single = t.dim() == 2
        if single:
            t = t.unsqueeze(0)
        t = t.contiguous()
        out = _io.empty(t.shape)
        ctx = nat.context()
        d = self._desc()
        nat.check(nat.library().redve_denoise(ctx, C.byref(d), t.shape[0], t.shape[1], t.shape[2],
                                              nat.dptr(t), nat.dptr(out)), ctx)
        out = out[0] if single else out
        return _io.to_host(out, from_np)


class Identity(_Native):
    """f(x) = x (denoisers.py:21-27); returns a copy."""

    name = "identity"
    kind = nat.DN_IDENTITY


class GaussianFilter(_Native):
    """Circular convolution with a normalised Gaussian (denoisers.py:30-46),
    evaluated as a direct periodic stencil with the reference's exact taps."""

    kind = nat.DN_CONV

    def __init__(self, std: float = 0.55, support: int = 5):
        self.std = float(std)
        self.support = int(support)
        self.psf: Psf = make_psf("gaussian", support, std)
        self.name = f"gaussian(std={std:g},support={support})"

    def _fill(self, d):
        d.ksize = self.psf.size
        d.taps = nat.hptr(self.psf.taps)


class Median3(_Native):
    """Periodic 3x3 median (BASELINE.json configs[1]); bit-exact order statistic,
    oracle ``scipy.ndimage.median_filter(size=3, mode="wrap")``."""

    name = "median3"
    kind = nat.DN_MEDIAN3
    linear = False


def denoise(spec, x):
    """denoisers.py:132-134."""
    from .imaging import as_image

    return spec(as_image(x))


def materialize_dense(spec, width: int, height: int) -> np.ndarray:
    """W with W @ vec(x) == vec(f(x)) for linear kinds (denoisers.py:137-154).

    Built in one batched call: the unit images are the columns of a batch."""
    if not getattr(spec, "linear", True):
        raise NotLinear(f"{type(spec).__name__} is input-dependent")
    n = width * height
    if n > 4096:
        raise ValueError(f"dense denoiser matrix capped at 4096 pixels, got {n}")
    basis = np.eye(n).reshape(n, height, width)
    if isinstance(spec, _Native):
        cols = np.asarray(spec(basis)).reshape(n, n)
    else:
        cols = np.stack([np.asarray(spec(basis[j])).ravel() for j in range(n)])
    return np.ascontiguousarray(cols.T)


BUILTIN_DENOISERS = {
    "identity": Identity,
    "gaussian": GaussianFilter,
    "median3": Median3,
}
