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

__all__ = ["Identity", "GaussianFilter", "Median3", "PatchWeighted", "FilterBank", "NotLinear", "materialize_dense",
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


class PatchWeighted(_Native):
    """Symmetric non-local-means smoother (denoisers.py:49-129).

    Same parameters and results as the reference; on the device the 20
    balancing sweeps update one scalar field D (w_o(p) = w0_o(p) D(p) D(p+o))
    instead of 49 maps, and only the 24 half-plane raw-weight maps are stored."""

    kind = nat.DN_PATCH
    linear = False

    def __init__(self, patch_radius: int = 1, search_radius: int = 3, h: float = 110.0,
                 balance_iters: int = 20, weight_dtype: str = "float64"):
        """``weight_dtype`` (not in the reference): storage of the raw-weight
        planes.  "float32" halves the sweeps' HBM traffic (BASELINE.json
        configs[2]/[4]: "fp32 with fp64 ... accumulation"); every product and
        sum stays fp64, the weights carry a 2^-24 relative rounding."""
        if patch_radius < 0 or search_radius < 1 or h <= 0 or balance_iters < 1:
            raise ValueError("need patch_radius >= 0, search_radius >= 1, h > 0, balance_iters >= 1")
        if weight_dtype not in ("float64", "float32"):
            raise ValueError("weight_dtype must be 'float64' or 'float32'")
        self.patch_radius = int(patch_radius)
        self.search_radius = int(search_radius)
        self.h = float(h)
        self.balance_iters = int(balance_iters)
        self.weight_dtype = weight_dtype
        self.name = f"patch_weighted(p={patch_radius},s={search_radius},h={h:g})"
        if weight_dtype == "float32":
            self.name += "[fp32 weights]"

    def _fill(self, d):
        d.patch_radius = self.patch_radius
        d.search_radius = self.search_radius
        d.balance_iters = self.balance_iters
        d.h = self.h
        d.weight_bits = 32 if self.weight_dtype == "float32" else 64

    def weight_maps(self, x):
        """(offsets, maps): the balanced weight of every search offset (denoisers.py:83-111)."""
        t, from_np = _io.to_device(x)
        if t.dim() != 2:
            raise ValueError("weight_maps takes one image")
        t = t.contiguous()
        r = self.search_radius
        side = 2 * r + 1
        maps = _io.empty((side * side,) + tuple(t.shape))
        ctx = nat.context()
        d = self._desc()
        nat.check(nat.library().redve_patch_weight_maps(ctx, C.byref(d), 1, t.shape[0], t.shape[1],
                                                        nat.dptr(t), nat.dptr(maps)), ctx)
        offsets = [(di, dj) for di in range(-r, r + 1) for dj in range(-r, r + 1)]
        m = _io.to_host(maps, True)
        return offsets, [m[k] for k in range(side * side)]

    @staticmethod
    def apply_maps(offsets, maps, z):
        """Apply a frozen weight field (denoisers.py:113-119)."""
        z = np.asarray(z, dtype=np.float64)
        out = np.zeros_like(z)
        for (di, dj), w in zip(offsets, maps):
            out += w * np.roll(z, (-di, -dj), axis=(0, 1))
        return out

    def linearized(self, x):
        """The denoiser with its weight field frozen at x (denoisers.py:121-124)."""
        offsets, maps = self.weight_maps(x)
        return lambda z: self.apply_maps(offsets, maps, np.asarray(z, dtype=np.float64))


def filter_bank_params(seed: int = 0, n_filters: int = 8, size: int = 5):
    """Seeded filter-bank parameters (BASELINE.json configs[3]: "parameters drawn
    from the seed"): zero-mean unit-norm k x k filters, influence scales in
    [10, 40], step tau = 0.5 / sum ||k_i||_1^2, drawn from PCG64(seed) in a fixed
    order (host-side setup, like the reference's seeded noise)."""
    gen = np.random.Generator(np.random.PCG64(seed))
    k = gen.standard_normal((n_filters, size, size))
    k -= k.mean(axis=(1, 2), keepdims=True)
    k /= np.sqrt((k**2).sum(axis=(1, 2), keepdims=True))
    scales = 10.0 + 30.0 * gen.random(n_filters)
    l1 = np.abs(k).sum(axis=(1, 2))
    tau = 0.5 / float((l1**2).sum())
    return np.ascontiguousarray(k), np.ascontiguousarray(scales), tau


class FilterBank(_Native):
    """One reaction-diffusion stage f(x) = x - tau sum_i k_i * phi_i(k_i (x) x),
    phi_i(z) = z / (1 + z^2/s_i^2) (the "reaction-diffusion filter bank with its
    influence nonlinearity" of BASELINE.json configs[3]; the reference has no
    such denoiser -- TNRD is out of its scope).  One fused CUDA
    stencil kernel per call."""

    kind = nat.DN_FILTERBANK
    linear = False

    def __init__(self, seed: int = 0, n_filters: int = 8, size: int = 5):
        if n_filters < 1 or size < 1 or size % 2 == 0:
            raise ValueError("need n_filters >= 1 and an odd filter size")
        self.seed, self.n_filters, self.size = int(seed), int(n_filters), int(size)
        self.k, self.s, self.tau = filter_bank_params(seed, n_filters, size)
        self.name = f"filter_bank(seed={seed},n={n_filters},k={size})"

    def _fill(self, d):
        d.n_filters = self.n_filters
        d.fsize = self.size
        d.filters = nat.hptr(self.k)
        d.scales = nat.hptr(self.s)
        d.tau = self.tau


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
    "patch-weighted": PatchWeighted,
    "median3": Median3,
    "filter-bank": FilterBank,
}
