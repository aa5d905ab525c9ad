"""Batched RED problems on the device -- the B200-native entry point.

``RedBatch(forward, ys, sigma, alpha, denoiser, references)`` is B reference
``RedObjective``s that share operator, denoiser, sigma and alpha
(objective.py:44-74) and differ in the measurement.  ``solve_batch`` runs
``solve`` (solvers.py:388-399) for all of them in one device-resident
schedule and returns per-image solutions and traces.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _io
from . import _native as nat
from .errors import CgNoConvergence, KernelTooLarge, NonFiniteIterate, ShapeMismatch

__all__ = ["RedBatch", "solve_batch", "BatchResult"]


def _operator_desc(forward):
    d = nat.OperatorDesc()
    d.kind = forward._kind
    d.ksize = forward.psf.size
    d.taps = nat.hptr(forward.psf.taps)
    d.factor = getattr(forward, "factor", 1)
    return d


def native_denoiser_desc(denoiser):
    """Descriptor of a built-in denoiser, or an EXTERNAL one for any callable."""
    if hasattr(denoiser, "_desc"):
        return denoiser._desc(), True
    d = nat.DenoiserDesc()
    d.kind = nat.DN_EXTERNAL
    return d, False


class RedBatch:
    """B RED objectives sharing (forward, sigma, alpha, denoiser) on one GPU."""

    def __init__(self, forward, ys, sigma: float, alpha: float, denoiser, references=None):
        if sigma <= 0:
            raise ValueError("sigma must be > 0")
        if alpha <= 0:
            raise ValueError("alpha must be > 0")
        if not hasattr(forward, "_kind"):
            raise TypeError("RedBatch needs a native operator (Blur / BlurDownsample)")
        self.forward = forward
        self.sigma = float(sigma)
        self.alpha = float(alpha)
        self.denoiser = denoiser
        yt, _ = _io.to_device(ys)
        if yt.dim() == 2:
            yt = yt.unsqueeze(0)
        if tuple(yt.shape[1:]) != tuple(forward.out_shape):
            raise ValueError(f"y shape {tuple(yt.shape[1:])} != operator output {forward.out_shape}")
        self.B = int(yt.shape[0])
        self.shape = tuple(forward.in_shape)
        self.y = yt.contiguous()
        self._y_src = ys  # x0 = y (the deblurring default, cli.py:362-363) reuses self.y
        self.ref = None
        if references is not None:
            rt, _ = _io.to_device(references)
            if rt.dim() == 2:
                rt = rt.unsqueeze(0)
            self.ref = rt.contiguous()
        self._dn_desc, self.native_denoiser = native_denoiser_desc(denoiser)
        self._op_desc = _operator_desc(forward)
        ctx = nat.context()
        h = C.c_void_p()
        H, W = self.shape
        rc = nat.library().redve_problem_create(
            ctx, C.byref(self._op_desc), C.byref(self._dn_desc), self.B, H, W, nat.dptr(self.y),
            self.sigma, self.alpha, nat.dptr(self.ref), C.byref(h))
        nat.check(rc, ctx)
        self._h = h
        self._ctx = ctx

    def set_measurements(self, ys, references=None):
        """New measurements (and PSNR references) for the same operator, denoiser,
        sigma and alpha: what a fresh ``RedBatch`` would compute (objective.py:61-74),
        in this one's device buffers and with its captured solve schedule."""
        yt, _ = _io.to_device(ys)
        if yt.dim() == 2:
            yt = yt.unsqueeze(0)
        if tuple(yt.shape) != tuple(self.y.shape):
            raise ShapeMismatch(f"expected measurements of shape {tuple(self.y.shape)}")
        rt = None
        if references is not None:
            rt, _ = _io.to_device(references)
            if rt.dim() == 2:
                rt = rt.unsqueeze(0)
            rt = rt.contiguous()
        if (rt is None) != (self.ref is None):
            raise ValueError("a RedBatch keeps its PSNR-reference mode (created "
                             f"{'without' if self.ref is None else 'with'} references)")
        yt = yt.contiguous()
        nat.context()  # bind the context to the caller's current stream
        nat.check(nat.library().redve_problem_set_measurements(self._h, nat.dptr(yt), nat.dptr(rt)),
                  self._ctx)
        self.y, self.ref, self._y_src = yt, rt, ys
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                nat.library().redve_problem_destroy(h)
            except Exception:  # pragma: no cover - interpreter teardown
                pass
            self._h = None

    # -- helpers ---------------------------------------------------------------
    def _ext_f(self, xt):
        """f(x) for a host-callable denoiser (the user's plug-in), on the device."""
        if self.native_denoiser:
            return None
        outs = [np.asarray(self.denoiser(xt[b].detach().cpu().numpy()), dtype=np.float64)
                for b in range(xt.shape[0])]
        ft, _ = _io.to_device(np.stack(outs))
        return ft

    def _batch_in(self, x):
        t, from_np = _io.to_device(x)
        single = t.dim() == 2 or (t.dim() == 1)
        H, W = self.shape
        t = t.reshape(-1, H, W).contiguous()
        if t.shape[0] != self.B:
            raise ShapeMismatch(f"expected {self.B} images of {self.shape}")
        return t, from_np, single

    # -- objective pieces (objective.py:78-121) ------------------------------------
    def fp_step(self, x):
        t, from_np, single = self._batch_in(x)
        f = self._ext_f(t)
        out = _io.empty(t.shape)
        nat.check(nat.library().redve_fp_step(self._h, nat.dptr(t), nat.dptr(out), nat.dptr(f)),
                  self._ctx)
        return out, from_np

    def fp_step_denoised(self, x):
        """(fp_step(x), f(x)) with f(x) as fused into the first FFT pass."""
        t, from_np, single = self._batch_in(x)
        out = _io.empty(t.shape)
        f = _io.empty(t.shape)
        nat.check(nat.library().redve_fp_step_denoised(self._h, nat.dptr(t), nat.dptr(out),
                                                       nat.dptr(f)), self._ctx)
        return out, f

    def gradient(self, x):
        """grad E(x) for every image (objective.py:90-93), on the device."""
        t, from_np, single = self._batch_in(x)
        f = self._ext_f(t)
        out = _io.empty(t.shape)
        nat.check(nat.library().redve_gradient(self._h, nat.dptr(t), nat.dptr(f), nat.dptr(out)),
                  self._ctx)
        return out, from_np

    def cost_terms(self, x):
        t, _, _ = self._batch_in(x)
        f = self._ext_f(t)
        cost = np.empty(self.B)
        fid = np.empty(self.B)
        reg = np.empty(self.B)
        ps = np.empty(self.B)
        nat.check(nat.library().redve_cost(self._h, nat.dptr(t), nat.dptr(f), nat.hptr(cost),
                                           nat.hptr(fid), nat.hptr(reg), nat.hptr(ps)), self._ctx)
        return cost, fid, reg, ps

    @property
    def device_solvable(self) -> bool:
        return self.native_denoiser

    @property
    def graph_captures(self) -> int:
        """How many times the device solve captured its CUDA graph."""
        return int(nat.library().redve_problem_graph_captures(self._h))

    # -- the device-resident solve ----------------------------------------------------
    def solve(self, x0, config, method=None):
        """Run ``config`` for every image; returns BatchResult (solutions on the device)."""
        from .solvers import SolveConfig  # noqa: F401  (type only)

        method = config.method if method is None else method
        if method not in nat.METHOD_CODES:
            raise ValueError(f"unknown method {method!r}")
        gradient = method in ("sd", "sd-ve", "nesterov")
        if gradient and (config.step_size is None or config.step_size <= 0):
            raise ValueError("this method needs a positive step_size")
        if x0 is self._y_src and tuple(self.y.shape[1:]) == self.shape:
            t = self.y  # the measurements already on the device: no second upload
        else:
            t, _, _ = self._batch_in(x0)  # finiteness of x0: checked on the device
        cfg = nat.SolveConfigC()
        cfg.method = nat.METHOD_CODES[method]
        cfg.ve_method = nat.VE_CODES[config.ve_method]
        cfg.m = config.m
        cfg.kappa = config.kappa
        cfg.max_inner_steps = config.max_inner_steps
        cfg.tol = config.tol
        cycling = method in ("fp-ve", "sd-ve")
        cfg.stabilization_iters = config.stabilization_iters if cycling else 0
        cfg.rank_tolerance = config.rank_tolerance
        cfg.step_size = float(config.step_size) if gradient else 0.0
        B = self.B
        cap = config.max_inner_steps + cfg.stabilization_iters
        clen = config.m + config.kappa + 1
        ccap = config.max_inner_steps // clen + 2
        res = BatchResult(B, cap, ccap)
        out = _io.empty(t.shape)
        nat.check(nat.library().redve_solve(self._h, C.byref(cfg), nat.dptr(t), nat.dptr(out),
                                            C.byref(res.c_struct())), self._ctx)
        res.x = out
        res.requested = config.ve_method
        return res


class BatchResult:
    """Per-image solutions (device tensor) + trace arrays (host)."""

    def __init__(self, B, cap, ccap):
        self.B, self.cap, self.ccap = B, cap, ccap
        f = lambda *s: np.full(s, np.nan)
        self.n_records = np.zeros(B, np.int32)
        self.step_norm = f(B, cap)
        self.cost = f(B, cap)
        self.psnr = f(B, cap)
        self.gamma_abs_sum = f(B, cap)
        self.elapsed_s = f(B, cap)
        self.n_cycles = np.zeros(B, np.int32)
        self.cycle_meta = np.zeros((B, ccap, 4), np.int32)
        self.cycle_stability = np.zeros((B, ccap))
        self.cycle_gamma = np.zeros((B, ccap, nat.MAXKP1))
        self.cycle_c = np.zeros((B, ccap, nat.MAXKP1))
        self.status = np.zeros(B, np.int32)
        self.returned_best = np.zeros(B, np.int32)
        self.cg_iters = np.zeros((B, cap), np.int32)
        self.x = None
        self.requested = None

    def c_struct(self):
        t = nat.TraceC()
        t.cap, t.ccap = self.cap, self.ccap
        ip = lambda a: nat.hptr(a, C.c_int32)
        t.n_records = ip(self.n_records)
        t.step_norm = nat.hptr(self.step_norm)
        t.cost = nat.hptr(self.cost)
        t.psnr = nat.hptr(self.psnr)
        t.gamma_abs_sum = nat.hptr(self.gamma_abs_sum)
        t.elapsed_s = nat.hptr(self.elapsed_s)
        t.n_cycles = ip(self.n_cycles)
        t.cycle_meta = ip(self.cycle_meta)
        t.cycle_stability = nat.hptr(self.cycle_stability)
        t.cycle_gamma = nat.hptr(self.cycle_gamma)
        t.cycle_c = nat.hptr(self.cycle_c)
        t.status = ip(self.status)
        t.returned_best = ip(self.returned_best)
        t.cg_iters = ip(self.cg_iters)
        self._keep = t
        return t

    def trace(self, b: int):
        from .solvers import trace_from_arrays

        n = int(self.n_records[b])
        return trace_from_arrays(n, self.step_norm[b], self.cost[b], self.psnr[b],
                                 self.gamma_abs_sum[b], self.elapsed_s[b], int(self.n_cycles[b]),
                                 self.cycle_meta[b], self.cycle_stability[b], self.cycle_gamma[b],
                                 self.cycle_c[b], self.requested)

    def raise_for(self, b: int):
        st = int(self.status[b])
        if st == nat.E_NONFINITE:
            tr = self.trace(b)
            raise NonFiniteIterate(f"iterate diverged at inner step {tr.inner_steps}", tr)
        if st == nat.E_CG:
            raise CgNoConvergence("CG residual above the abort threshold")


def solve_batch(batch: RedBatch, x0, config):
    """Solve every problem of ``batch``; returns (solutions [B, H, W] CUDA tensor,
    list of IterationTrace).  Per-image failures raise like the reference."""
    res = batch.solve(x0, config)
    for b in range(batch.B):
        res.raise_for(b)
    return res.x, [res.trace(b) for b in range(batch.B)]
