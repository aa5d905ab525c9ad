"""CPU stand-in for spatial.NativeSlabOps (TEST INFRASTRUCTURE: built on the
oracle, only used by the gloo tests of the distributed driver's plumbing).

Tensors are torch CPU fp64; the arithmetic is numpy restating the oracle's
operators on the extended slab (periodic within the buffer, exact on the
interior because the halo covers every reach)."""

import numpy as np
import torch

from oracle import redve_ref as R

VE = {"mpe": 0, "rre": 1, "svdmpe": 2}


class _Res:
    def __init__(self):
        self.converged = 0
        self.extrapolated = 0
        self.kappa_used = 0
        self.method = 0
        self.fallback = 0
        self.stability_sum = 0.0
        self.gamma = [0.0] * 12
        self.c = [0.0] * 12


def _weights_from_r(r, e, method):
    """extrapolation.py:359-386 on a given R and rank (restated via the oracle)."""
    res = _Res()
    n = r.shape[0]
    kappa = n - 1
    if e == n:
        w, used = None, method
        if method == "mpe":
            w = R._annihilate(r, kappa)
        elif method == "svdmpe":
            w = R.weights_svdmpe(r)
        if method == "rre" or w is None:
            res.fallback = int(method != "rre")
            w, used = R.weights_rre(r), "rre"
        ke = kappa
    else:
        w = R._annihilate(r, e)
        if w is None:
            return res, np.zeros(12)
        used, ke = method, e
    c, g = w
    res.extrapolated = 1
    res.kappa_used = ke
    res.method = VE[used]
    res.stability_sum = float(np.abs(g).sum())
    res.gamma[: ke + 1] = list(g)
    res.c[: ke + 1] = list(c)
    xi = np.zeros(12)
    xi[:ke] = 1.0 - np.cumsum(g[:ke])
    return res, xi


class CpuSlabOps:
    def __init__(self, taps, factor, sigma, alpha, denoiser):
        self.taps = np.asarray(taps, dtype=np.float64)
        self.s, self.sigma, self.alpha, self.denoiser = factor, sigma, alpha, denoiser

    def tensor(self, a):
        return torch.from_numpy(np.array(a, dtype=np.float64))

    def zeros(self, shape):
        return torch.zeros(shape, dtype=torch.float64)

    def host(self, t):
        return t.numpy().copy()

    def copy(self, t):
        return t.clone()

    def _blur(self, shape):
        return R.CirculantBlur(self.taps, shape)

    def _mask(self, shape, row0, Hg):
        m = np.zeros(shape)
        for u in range(shape[0]):
            if ((row0 + u) % Hg) % self.s == 0:
                m[u, :: self.s] = 1.0
        return m

    def denoise(self, x_ext):
        return torch.from_numpy(np.asarray(self.denoiser(x_ext.numpy()), dtype=np.float64))

    def correlate(self, z_ext, scale):
        return torch.from_numpy(self._blur(z_ext.shape).adjoint(z_ext.numpy()) * scale)

    def normal_matvec(self, w_ext, row0, Hg):
        b = self._blur(w_ext.shape)
        w = w_ext.numpy()
        z = b.apply(w) * self._mask(w.shape, row0, Hg)
        return torch.from_numpy(b.adjoint(z) / self.sigma**2 + self.alpha * w)

    def dot(self, x, y):
        return float(np.dot(x.numpy().ravel(), y.numpy().ravel()))

    def dist2(self, x, y):
        d = (x.numpy() - y.numpy()).ravel()
        return float(np.dot(d, d))

    def axpby(self, a, x, b, y):
        y.copy_(torch.from_numpy(a * x.numpy() + b * y.numpy()))

    def fidelity(self, x_ext, yup_ext, row0, Hg, halo, rows):
        x = x_ext.numpy()
        d = (self._blur(x.shape).apply(x) - yup_ext.numpy()) * self._mask(x.shape, row0, Hg)
        d = d[halo: halo + rows]
        return float(np.vdot(d, d))

    def window_gram(self, window):
        w = window.numpy().reshape(window.shape[0], -1)
        u = np.diff(w, axis=0)
        return u @ u.T

    def decide(self, G, method, rank_tol):
        n = G.shape[0]
        if not np.all(np.isfinite(G)):
            return _Res(), np.zeros(12), False
        if G[0, 0] <= 0 or np.sqrt(G[0, 0]) < 1e-300:
            res = _Res()
            res.converged = 1
            return res, np.zeros(12), False
        try:
            r = np.linalg.cholesky(G).T
        except np.linalg.LinAlgError:
            return _Res(), np.zeros(12), True
        thr = max(1e-6, 1e3 * rank_tol)
        if np.any(np.diag(r)[1:] < thr * r[0, 0]):
            return _Res(), np.zeros(12), True
        res, xi = _weights_from_r(r, n, method)
        return res, xi, False

    def decide_r(self, Rm, rank, method):
        return _weights_from_r(np.asarray(Rm), rank, method)

    def combine(self, window, ke, xi):
        w = window.numpy()
        out = w[0].copy()
        for j in range(ke):
            out = out + xi[j] * (w[j + 1] - w[j])
        return torch.from_numpy(out)

    def stack(self, vs):
        return torch.stack(vs).contiguous()
