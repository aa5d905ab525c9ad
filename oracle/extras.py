"""Oracles for the BASELINE.json plug-ins the reference does not contain (TEST ORACLE).

Test infrastructure only (see ``oracle/__init__.py``).  They plug into the
reference's callable-denoiser protocol (``denoisers.py:1-8``; any
``f(x: ndarray[H, W]) -> ndarray[H, W]``), so ``redve_ref.Red`` and the real
reference ``RedObjective`` accept them unchanged.

* ``median3``  -- periodic 3x3 median.  Pinned bit-exact against
  ``scipy.ndimage.median_filter(size=3, mode="wrap")`` in tests; the roll
  formulation below is an independent restatement.
* ``FilterBank`` -- one seeded reaction-diffusion (Field-of-Experts gradient)
  stage  f(x) = x - tau * sum_i  kbar_i * phi(k_i * x),  phi(z) = z/(1+z^2/s^2).
  PARITY UNPINNED: no reference implementation exists.
"""

from __future__ import annotations

import numpy as np


def median3(x):
    """Periodic 3x3 median via the 9 rolled copies (median of 9 = 5th order stat)."""
    x = np.asarray(x, dtype=np.float64)
    stack = np.stack([np.roll(x, (a, b), axis=(0, 1)) for a in (-1, 0, 1) for b in (-1, 0, 1)])
    return np.sort(stack, axis=0)[4]


def filter_bank_params(seed: int = 0, n_filters: int = 8, size: int = 5):
    """Seeded filter-bank parameters: zero-mean k x k filters with unit l2 norm,
    per-filter influence scales s_i in [10, 40], step tau = 0.5/sum ||k_i||_1^2.

    Drawn from ``numpy.random.Generator(PCG64(seed))`` in a fixed order so the
    GPU path and the oracle share bit-identical parameters."""
    gen = np.random.Generator(np.random.PCG64(seed))
    k = gen.standard_normal((n_filters, size, size))
    k -= k.mean(axis=(1, 2), keepdims=True)
    k /= np.sqrt((k**2).sum(axis=(1, 2), keepdims=True))
    scales = 10.0 + 30.0 * gen.random(n_filters)
    l1 = np.abs(k).sum(axis=(1, 2))
    tau = 0.5 / float((l1**2).sum())
    return k, scales, tau


def _corr_periodic(x, k):
    """y[i,j] = sum_{a,b} k[a,b] x[i+a-r, j+b-r] (correlation, periodic)."""
    r = k.shape[0] // 2
    y = np.zeros_like(x)
    for a in range(k.shape[0]):
        for b in range(k.shape[1]):
            y += k[a, b] * np.roll(x, (r - a, r - b), axis=(0, 1))
    return y


def _conv_periodic(x, k):
    """Adjoint of ``_corr_periodic``: y[i,j] = sum_{a,b} k[a,b] x[i-a+r, j-b+r]."""
    r = k.shape[0] // 2
    y = np.zeros_like(x)
    for a in range(k.shape[0]):
        for b in range(k.shape[1]):
            y += k[a, b] * np.roll(x, (a - r, b - r), axis=(0, 1))
    return y


class FilterBank:
    """Seeded reaction-diffusion stage (oracle for the ``RD`` CUDA denoiser)."""

    def __init__(self, seed: int = 0, n_filters: int = 8, size: int = 5):
        self.k, self.s, self.tau = filter_bank_params(seed, n_filters, size)

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        acc = np.zeros_like(x)
        for k, s in zip(self.k, self.s):
            z = _corr_periodic(x, k)
            acc += _conv_periodic(z / (1.0 + (z * z) / (s * s)), k)
        return x - self.tau * acc
