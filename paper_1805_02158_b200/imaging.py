"""Images, PSFs and degradation operators -- drop-in for ``redve.imaging``.

``Blur`` / ``BlurDownsample`` keep the reference's constructor, attributes and
``apply`` / ``adjoint`` contract (imaging.py:147-204); the arithmetic runs in
libredve_b200 as direct periodic stencils (conv / correlate / decimate /
zero-fill), not FFTs.  Inputs may be numpy arrays (copied to and from the
GPU) or CUDA tensors, single images ``[H, W]`` or batches ``[B, H, W]``.

Host-side input synthesis stays on the host exactly like the reference
(``gaussian_noise`` / ``degrade`` / ``synthetic_image``; SURVEY.md section
8a row A21): identical seeds give bit-identical noise on both paths.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _io
from . import _native as nat
from .errors import InvalidSize, KernelTooLarge, ShapeMismatch

__all__ = [
    "Psf", "make_psf", "Blur", "BlurDownsample", "InvalidSize", "KernelTooLarge",
    "ShapeMismatch", "as_image", "gaussian_noise", "degrade", "psnr", "synthetic_image",
]


def as_image(x) -> np.ndarray:
    """Finite 2-D float64 image (imaging.py:31-38)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ShapeMismatch(f"expected a 2-D image, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError("image contains non-finite entries")
    return a


@dataclass(frozen=True)
class Psf:
    """k x k kernel with a centred anchor (imaging.py:46-68)."""

    size: int
    taps: np.ndarray
    kind: str = "custom"

    def __post_init__(self):
        if self.size < 1 or self.size % 2 == 0:
            raise InvalidSize(f"PSF size must be odd and >= 1, got {self.size}")
        taps = np.ascontiguousarray(np.asarray(self.taps, dtype=np.float64))
        if taps.shape != (self.size, self.size):
            raise InvalidSize(f"taps shape {taps.shape} != ({self.size}, {self.size})")
        object.__setattr__(self, "taps", taps)

    @property
    def radius(self) -> int:
        return self.size // 2


def make_psf(kind: str, size: int, std: float | None = None) -> Psf:
    """Normalised uniform or Gaussian kernel (imaging.py:71-92)."""
    if size < 1 or size % 2 == 0:
        raise InvalidSize(f"PSF size must be odd and >= 1, got {size}")
    if kind == "uniform":
        return Psf(size, np.full((size, size), 1.0 / size**2), "uniform")
    if kind == "gaussian":
        if std is None or std <= 0:
            raise InvalidSize("gaussian PSF needs std > 0")
        half = size // 2
        axis = np.arange(-half, half + 1, dtype=np.float64)
        rr, cc = np.meshgrid(axis, axis, indexing="ij")
        taps = np.exp(-(rr**2 + cc**2) / (2.0 * std**2))
        return Psf(size, taps / taps.sum(), "gaussian")
    raise InvalidSize(f"unknown PSF kind {kind!r}")


# ---------------------------------------------------------------- DFT helpers
# (imaging.py:100-145).  Host arrays follow numpy's convention exactly, as the
# reference; device tensors stay on the device (cuFFT through torch) -- these
# are utilities, the solver's transforms are fourier.cu's fused kernels.


def dft2(image):
    """2-D DFT, numpy "backward" convention (idft2(dft2(x)) == x)."""
    if _io.is_tensor(image):
        return _io.torch_mod().fft.fft2(image)
    return np.fft.fft2(image)


def idft2(spectrum):
    """Inverse of :func:`dft2`; the real part."""
    if _io.is_tensor(spectrum):
        return _io.torch_mod().fft.ifft2(spectrum).real
    return np.fft.ifft2(spectrum).real


def embed_psf(psf: "Psf", shape) -> np.ndarray:
    """The kernel in a full-size array with its anchor at (0, 0)."""
    h, w = shape
    if psf.size > min(h, w):
        raise KernelTooLarge(f"{psf.size}x{psf.size} PSF on a {h}x{w} image")
    full = np.zeros(shape)
    full[: psf.size, : psf.size] = psf.taps
    return np.roll(full, (-psf.radius, -psf.radius), axis=(0, 1))


def psf_spectrum(psf: "Psf", shape) -> np.ndarray:
    """Transfer function of circular convolution with the kernel."""
    return dft2(embed_psf(psf, shape))


def convolve_circular(image, psf: "Psf"):
    """Circular convolution of an image with a kernel (imaging.py:132-145),
    computed by the device stencil (same sum as the reference's DFT product)."""
    shape = tuple(np.shape(image))[-2:]
    return Blur(psf, shape).apply(image)


def _batched(x, shape):
    t, from_np = _io.to_device(x)
    single = t.dim() == 2
    if single:
        t = t.unsqueeze(0)
    if t.dim() != 3 or tuple(t.shape[1:]) != tuple(shape):
        raise ShapeMismatch(f"expected {tuple(shape)}, got {tuple(x.shape)}")
    return t.contiguous(), from_np, single


class _Operator:
    is_circulant = False

    def _desc(self):
        d = nat.OperatorDesc()
        d.kind = self._kind
        d.ksize = self.psf.size
        d.taps = nat.hptr(self.psf.taps)
        d.factor = getattr(self, "factor", 1)
        return d

    def _run(self, fn, x, in_shape, out_shape):
        t, from_np, single = _batched(x, in_shape)
        out = _io.empty((t.shape[0],) + tuple(out_shape))
        ctx = nat.context()
        d = self._desc()
        nat.check(fn(ctx, C.byref(d), t.shape[0], self.in_shape[0], self.in_shape[1],
                     nat.dptr(t), nat.dptr(out)), ctx)
        out = out[0] if single else out
        return _io.to_host(out, from_np)

    @property
    def spectrum(self) -> np.ndarray:
        """psf_spectrum of the blur on the input grid (imaging.py:165, 191)."""
        sp = getattr(self, "_spectrum", None)
        if sp is None:
            sp = psf_spectrum(self.psf, self.in_shape)
            self._spectrum = sp
        return sp

    def apply(self, x):
        return self._run(nat.library().redve_operator_apply, x, self.in_shape, self.out_shape)

    def adjoint(self, z):
        return self._run(nat.library().redve_operator_adjoint, z, self.out_shape, self.in_shape)


class Blur(_Operator):
    """Circular convolution H and its adjoint (imaging.py:147-170)."""

    is_circulant = True
    _kind = nat.OP_BLUR

    def __init__(self, psf: Psf, shape):
        h, w = shape
        if psf.size > min(h, w):
            raise KernelTooLarge(f"{psf.size}x{psf.size} PSF on a {h}x{w} image")
        self.psf = psf
        self.in_shape = tuple(shape)
        self.out_shape = tuple(shape)
        self.factor = 1


class BlurDownsample(_Operator):
    """Blur then keep indices == 0 mod factor (imaging.py:173-204)."""

    is_circulant = False
    _kind = nat.OP_BLUR_DOWNSAMPLE

    def __init__(self, psf: Psf, factor: int, shape):
        if factor < 1:
            raise InvalidSize(f"downsample factor must be >= 1, got {factor}")
        h, w = shape
        if psf.size > min(h, w):
            raise KernelTooLarge(f"{psf.size}x{psf.size} PSF on a {h}x{w} image")
        self.psf = psf
        self.factor = int(factor)
        self.in_shape = tuple(shape)
        self.out_shape = (-(-h // self.factor), -(-w // self.factor))


def gaussian_noise(shape, sigma: float, seed: int) -> np.ndarray:
    """Seeded PCG64 + Box-Muller field, bit-identical to imaging.py:207-218 (host)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = int(np.prod(shape))
    u1 = 1.0 - rng.random(n)
    u2 = rng.random(n)
    return sigma * (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).reshape(shape)


def degrade(image, op, sigma: float, seed: int) -> np.ndarray:
    """H x + e with seeded noise (imaging.py:221-231); H x on the GPU."""
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    clean = op.apply(as_image(image))
    if sigma == 0:
        return clean
    return clean + gaussian_noise(clean.shape, sigma, seed)


def psnr(x, reference) -> float:
    """PSNR with peak 255 (imaging.py:234-248); host metric utility."""
    x = np.asarray(x, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    if x.shape != reference.shape:
        raise ShapeMismatch(f"{x.shape} vs {reference.shape}")
    mse = np.mean((x - reference) ** 2)
    if mse == 0.0:
        return np.inf
    if not np.isfinite(mse):
        return -np.inf
    return 10.0 * np.log10(255.0**2 / mse)


def synthetic_image(height: int, width: int | None = None) -> np.ndarray:
    """The reference's deterministic test scene (imaging.py:251-270), host-side."""
    width = height if width is None else width
    ii, jj = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    v = ii / max(height - 1, 1)
    u = jj / max(width - 1, 1)
    img = 110.0 + 60.0 * np.sin(2 * np.pi * (1.5 * u + 0.5)) * np.cos(2 * np.pi * v)
    img[((u - 0.3) ** 2 + (v - 0.35) ** 2) < 0.04] = 220.0
    square = (np.abs(u - 0.72) < 0.12) & (np.abs(v - 0.68) < 0.12)
    img[square] = 35.0
    stripes = (np.abs(u + v - 1.35) < 0.18) & ~square
    img[stripes] += 45.0 * np.sin(24 * np.pi * (u - v))[stripes]
    return np.clip(img, 5.0, 250.0)
