"""Spatially partitioned super-resolution solve (BASELINE.json configs[4]).

One huge image is split into row slabs, one per rank (one process per GPU).
Every rank keeps its slab plus ``halo`` rows on each side (periodic ring of
neighbours: the last slab's bottom halo is the first slab's top rows, the
reference's all-periodic boundary, imaging.py:8-9).  Per fixed-point step:

* one halo exchange of x (reach of the denoiser and of the normal operator);
  the CG direction p exchanges only the normal operator's reach (2r rows);
* the denoiser on the extended slab (its result is exact on the interior
  rows because the halo covers the denoiser's reach);
* conjugate gradients with scipy's semantics (iterative.py:311-430) on the
  interior, the normal operator applied to the extended search direction
  after a halo exchange of p, every inner product allreduced;
* the step norm, cost terms and the VE Gram allreduced, so every rank takes
  the same decisions (termination, cadence, best iterate, extrapolation).

The algebra runs in libredve_b200 slab primitives (``NativeSlabOps``); the
collectives go through ``torch.distributed`` (NCCL on GPUs, gloo on CPU).
SURVEY.md section 8e.  Driver semantics follow solvers.py:206-385.
"""

from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np

from . import _io
from . import _native as nat
from .errors import CgNoConvergence, NonFiniteIterate
from .extrapolation import METHODS
from .shard import shard_bounds
from .solvers import IterationTrace, TraceRecord
from . import extrapolation as ve

CG_RTOL, CG_MAXITER, CG_ABORT = 1e-6, 200, 1e-4  # objective.py:35-37
DENSE_LOG_LIMIT = 128 * 128


# ----------------------------------------------------------------------------- layout
class SlabLayout:
    """Row slab of rank ``rank``: HR rows [start, stop), LR-aligned boundaries."""

    def __init__(self, H: int, W: int, factor: int, world: int, rank: int, halo: int):
        n_lr = -(-H // factor)
        lo, hi = shard_bounds(n_lr, world, rank)
        self.start = lo * factor
        self.stop = H if rank == world - 1 else hi * factor
        self.rows = self.stop - self.start
        self.H, self.W, self.factor, self.halo = H, W, factor, halo
        if self.rows < halo:
            raise ValueError(f"slab of {self.rows} rows is thinner than the halo ({halo})")
        self.Hext = self.rows + 2 * halo
        self.row0 = (self.start - halo) % H  # global row of extended row 0

    def ext_rows(self):
        return [(self.row0 + u) % self.H for u in range(self.Hext)]


def denoiser_reach(denoiser) -> int:
    name = type(denoiser).__name__
    if name == "PatchWeighted":
        pr, sr, it = denoiser.patch_radius, denoiser.search_radius, denoiser.balance_iters
        return pr + 2 * sr + sr * (it + 1)
    if name == "Median3":
        return 1
    if name == "GaussianFilter":
        return denoiser.psf.radius
    if name == "FilterBank":
        return 2 * (denoiser.size // 2)
    if name == "Identity":
        return 0
    raise TypeError(f"no reach known for denoiser {name}")


# ----------------------------------------------------------------------------- comm
class TorchComm:
    """Halo exchange + scalar allreduce over torch.distributed (or a single rank)."""

    def __init__(self, group=None, device="cpu"):
        import torch.distributed as dist

        self.dist = dist if (dist.is_available() and dist.is_initialized()) else None
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.group = group
        self.device = device  # where collective buffers live ("cpu" for gloo)

    def allreduce(self, vals):
        import torch

        if self.world == 1:
            return [float(v) for v in vals]
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t, group=self.group)
        return [float(v) for v in t.cpu().tolist()]

    def exchange(self, ext, halo: int, rows: int):
        """Fill ext[:halo] / ext[halo+rows:] (row-major [Hext, W] tensor) from the ring."""
        import torch

        if halo == 0:
            return
        top_int = ext[halo: 2 * halo]              # my first interior rows
        bot_int = ext[rows: rows + halo]            # my last interior rows
        if self.world == 1:
            ext[:halo].copy_(bot_int)
            ext[halo + rows:].copy_(top_int)
            return
        prev = (self.rank - 1) % self.world
        nxt = (self.rank + 1) % self.world
        dev = self.device
        send_bot = bot_int.contiguous().to(dev)
        send_top = top_int.contiguous().to(dev)
        recv_top = torch.empty_like(send_top)
        recv_bot = torch.empty_like(send_bot)
        P2P = self.dist.P2POp
        ops = [P2P(self.dist.isend, send_bot, nxt, self.group),
               P2P(self.dist.isend, send_top, prev, self.group),
               P2P(self.dist.irecv, recv_top, prev, self.group),
               P2P(self.dist.irecv, recv_bot, nxt, self.group)]
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        ext[:halo].copy_(recv_top)
        ext[halo + rows:].copy_(recv_bot)


class PeerComm(TorchComm):
    """Halo exchange by direct stores into the neighbours' buffers.

    Each rank's extended buffers are mapped into its two ring neighbours over
    CUDA IPC once (handles swapped with one all_gather per buffer); from then
    on ``push`` is ONE kernel (``redve_halo_push``) that writes the slab into
    this rank's buffer and, in the same pass, its edge rows straight into the
    previous rank's bottom halo and the next rank's top halo — over NVLink
    between GPUs, no staging copies and no send/recv.  Ordering: every rank
    drains its stream and meets a barrier before the stores (the neighbours are
    done reading their halos) and again after them (its own halos are full).
    Allreduces stay on torch.distributed (``device``: "cuda" for NCCL, "cpu"
    for gloo).
    """

    def _register(self, ext, halo: int, rows: int):
        """(prev_bot, next_top) views for ``ext``, mapped on first use.  The
        mapping lives on the buffer itself, so it is released with it."""
        import pickle
        from multiprocessing.reduction import ForkingPickler

        import torch
        import torch.multiprocessing  # noqa: F401  (registers the CUDA IPC reductions)

        ent = getattr(ext, "_redve_peer", None)
        if ent is not None and ent[0] == (halo, rows):
            return ent[1], ent[2]
        if self.world == 1:
            ent = ((halo, rows), ext[halo + rows:], ext[:halo])
        else:
            mine = (bytes(ForkingPickler.dumps(ext)), rows, ext.device.index)
            allv = [None] * self.world
            self.dist.all_gather_object(allv, mine, group=self.group)
            prev = (self.rank - 1) % self.world
            nxt = (self.rank + 1) % self.world
            lib, ctx = nat.library(), nat.context()
            for peer in {prev, nxt}:
                dev = allv[peer][2]
                if dev != ext.device.index:
                    nat.check(lib.redve_enable_peer_access(ctx, dev), ctx)
            pext = pickle.loads(allv[prev][0])
            next_ext = pext if nxt == prev else pickle.loads(allv[nxt][0])
            rp = allv[prev][1]
            ent = ((halo, rows), pext[halo + rp: 2 * halo + rp], next_ext[:halo])
            torch.cuda.current_stream().synchronize()
        ext._redve_peer = ent
        return ent[1], ent[2]

    def _fence(self):
        import torch

        if self.world > 1:  # one rank: stream order is enough
            torch.cuda.current_stream().synchronize()
            self.dist.barrier(group=self.group)

    def push(self, ext, x, halo: int, rows: int):
        """ext[halo:halo+rows] <- x, and the ring's halos of every rank filled."""
        if halo == 0:
            ext[:rows].copy_(x)
            return
        prev_bot, next_top = self._register(ext, halo, rows)
        x = x.contiguous()
        lib, ctx = nat.library(), nat.context()
        self._fence()
        nat.check(lib.redve_halo_push(ctx, rows, ext.shape[1], halo, nat.dptr(x), nat.dptr(ext),
                                      nat.dptr(prev_bot), nat.dptr(next_top)), ctx)
        self._fence()

    def exchange(self, ext, halo: int, rows: int):
        self.push(ext, ext[halo: halo + rows].clone(), halo, rows)


# ----------------------------------------------------------------------------- local ops
class NativeSlabOps:
    """Slab algebra in libredve_b200 (device tensors)."""

    def __init__(self, forward, sigma, alpha, denoiser):
        import torch

        self.torch = torch
        self.forward, self.sigma, self.alpha, self.denoiser = forward, sigma, alpha, denoiser
        self.lib = nat.library()
        self.ctx = nat.context()
        d = nat.OperatorDesc()
        d.kind = nat.OP_BLUR_DOWNSAMPLE
        d.ksize = forward.psf.size
        d.taps = nat.hptr(forward.psf.taps)
        d.factor = forward.factor
        self.op = d
        b = nat.OperatorDesc()
        b.kind = nat.OP_BLUR
        b.ksize = forward.psf.size
        b.taps = nat.hptr(forward.psf.taps)
        b.factor = 1
        self.blur = b

    def tensor(self, a):
        if isinstance(a, self.torch.Tensor):  # host rows, possibly page-locked: asynchronous when pinned
            return a.to(device="cuda", dtype=self.torch.float64, non_blocking=a.is_pinned()).contiguous()
        return self.torch.as_tensor(np.ascontiguousarray(a), dtype=self.torch.float64).cuda()

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.float64, device="cuda")

    def host(self, t):
        from . import _io

        return _io.host_array(t)

    def copy(self, t):
        return t.clone()

    def denoise(self, x_ext):
        return self.denoiser(x_ext)

    def correlate(self, z_ext, scale):
        out = self.zeros(z_ext.shape)
        nat.check(self.lib.redve_operator_adjoint(self.ctx, C.byref(self.blur), 1, z_ext.shape[0],
                                                  z_ext.shape[1], nat.dptr(z_ext), nat.dptr(out)),
                  self.ctx)
        self.axpby(0.0, out, scale, out)
        return out

    def normal_matvec(self, w_ext, row0, Hg):
        out = self.zeros(w_ext.shape)
        nat.check(self.lib.redve_sr_normal_matvec(self.ctx, C.byref(self.op), self.sigma, self.alpha,
                                                  w_ext.shape[0], w_ext.shape[1], row0, Hg,
                                                  nat.dptr(w_ext), nat.dptr(out)), self.ctx)
        return out

    def _red(self, fn, x, y):
        v = C.c_double()
        nat.check(fn(self.ctx, x.numel(), nat.dptr(x), nat.dptr(y), C.byref(v)), self.ctx)
        return v.value

    def dot(self, x, y):
        return self._red(self.lib.redve_vec_dot, x.contiguous(), y.contiguous())

    def dist2(self, x, y):
        return self._red(self.lib.redve_vec_dist2, x.contiguous(), y.contiguous())

    def axpby(self, a, x, b, y):
        nat.check(self.lib.redve_vec_axpby(self.ctx, y.numel(), float(a), nat.dptr(x), float(b),
                                           nat.dptr(y)), self.ctx)

    def fidelity(self, x_ext, yup_ext, row0, Hg, halo, rows):
        v = C.c_double()
        nat.check(self.lib.redve_sr_fidelity(self.ctx, C.byref(self.op), x_ext.shape[0],
                                             x_ext.shape[1], row0, Hg, halo, rows,
                                             nat.dptr(x_ext), nat.dptr(yup_ext), C.byref(v)),
                  self.ctx)
        return v.value

    def window_gram(self, window):
        rows = window.shape[0]
        G = np.zeros((rows - 1, rows - 1))
        nat.check(self.lib.redve_window_gram(self.ctx, rows, window[0].numel(), nat.dptr(window),
                                             nat.hptr(G)), self.ctx)
        return G

    def decide(self, G, method, rank_tol):
        kp1 = G.shape[0]
        res = nat.VeResultC()
        xi = np.zeros(12)
        need = C.c_int()
        G = np.ascontiguousarray(G)
        nat.check(self.lib.redve_ve_decide(self.ctx, kp1, nat.hptr(G), nat.VE_CODES[method],
                                           rank_tol, C.byref(res), nat.hptr(xi), C.byref(need)),
                  self.ctx)
        return res, xi, bool(need.value)

    def decide_r(self, R, rank, method):
        kp1 = R.shape[0]
        res = nat.VeResultC()
        xi = np.zeros(12)
        R = np.ascontiguousarray(R)
        nat.check(self.lib.redve_ve_decide_r(self.ctx, kp1, nat.hptr(R), rank, nat.VE_CODES[method],
                                             C.byref(res), nat.hptr(xi)), self.ctx)
        return res, xi

    def combine(self, window, ke, xi):
        out = self.zeros(window.shape[1:])
        xi = np.ascontiguousarray(xi[:ke])
        nat.check(self.lib.redve_window_combine(self.ctx, window.shape[0], window[0].numel(),
                                                nat.dptr(window), ke, nat.hptr(xi),
                                                nat.dptr(out)), self.ctx)
        return out

    def stack(self, vs):
        return self.torch.stack(vs).contiguous()


# ----------------------------------------------------------------------------- driver
class PinnedHost:
    """A host image held in page-locked memory.  ``SpatialProblem`` (y,
    reference) and ``solve_spatial`` (x0, ``out``) take it wherever they take a
    numpy image; the slab's rows then cross the bus at PCIe rate, asynchronously
    on the solver's stream, instead of through pageable staging (8192^2 fp64:
    ~100 ms per direction pageable against ~11 ms pinned).  Pin once, reuse."""

    def __init__(self, a=None, shape=None):
        torch = _io.torch_mod()
        if a is None:
            t = torch.empty(tuple(shape), dtype=torch.float64)
        elif _io.is_tensor(a):
            t = a.detach().to(device="cpu", dtype=torch.float64).contiguous()
        else:
            t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
        self.t = t if t.is_pinned() else t.pin_memory()

    @property
    def shape(self):
        return tuple(self.t.shape)

    def numpy(self):
        return self.t.numpy()


class SpatialProblem:
    """One SR problem split across the ranks of ``comm`` (RedObjective over slabs)."""

    def __init__(self, forward, y, sigma, alpha, denoiser, comm=None, ops=None, reference=None,
                 reach=None):
        if sigma <= 0 or alpha <= 0:
            raise ValueError("sigma, alpha must be > 0")
        self.comm = comm or TorchComm()
        self.ops = ops or NativeSlabOps(forward, sigma, alpha, denoiser)
        H, W = forward.in_shape
        self.H, self.W, self.s = H, W, forward.factor
        self.sigma, self.alpha = float(sigma), float(alpha)
        r = forward.psf.radius
        halo = max(denoiser_reach(denoiser) if reach is None else int(reach), 2 * r)
        self.lay = SlabLayout(H, W, self.s, self.comm.world, self.comm.rank, halo)
        # the normal operator's reach (H^T H: 2r rows): the CG direction p only
        # needs these rows from the neighbours, not the denoiser's halo
        self.op_lay = SlabLayout(H, W, self.s, self.comm.world, self.comm.rank, 2 * r)
        lay = self.lay
        y = y.numpy() if isinstance(y, PinnedHost) else np.asarray(y, dtype=np.float64)
        # zero-filled upsampling of the slab's measurement rows, built on the
        # device: only the LR rows the slab touches cross the bus
        rows = [(u, g // self.s) for u, g in enumerate(lay.ext_rows()) if g % self.s == 0]
        yup = self.ops.zeros((lay.Hext, W))
        if rows:
            yup[[u for u, _ in rows], ::self.s] = self.ops.tensor(y[[g for _, g in rows]])
        self.yup = yup
        self.hty = self.ops.correlate(self.yup, 1.0 / self.sigma**2)[lay.halo: lay.halo + lay.rows]
        self.ref = None if reference is None else self._rows_to_device(reference)
        self.N = H * W
        self._ext = {}
        self._fcache = None  # (x, x._version, f(x))

    # -- helpers
    def _rows_to_device(self, image):
        """This rank's rows of a host image (numpy or PinnedHost) on the device."""
        if isinstance(image, PinnedHost):
            return self.ops.tensor(image.t[self.lay.start: self.lay.stop])
        return self.ops.tensor(np.asarray(image, dtype=np.float64)[self.lay.start: self.lay.stop])

    def slab(self, x_global):
        """This rank's rows of a host image (a device tensor is taken as the slab itself)."""
        if isinstance(x_global, PinnedHost):
            return self._rows_to_device(x_global)
        if hasattr(x_global, "is_cuda") or hasattr(x_global, "clone"):
            if tuple(x_global.shape) != (self.lay.rows, self.W):
                raise ValueError(f"slab tensor must be {(self.lay.rows, self.W)}")
            return x_global.clone()
        return self.ops.tensor(np.asarray(x_global, dtype=np.float64)[self.lay.start: self.lay.stop])

    def extend(self, x, slot="x", lay=None):
        """x with its halos (``lay``: the denoiser's by default) from the ring, in
        a persistent per-slot buffer."""
        lay = lay or self.lay
        ext = self._ext.get(slot)
        if ext is None:
            ext = self._ext[slot] = self.ops.zeros((lay.Hext, self.W))
        if hasattr(self.comm, "push"):  # one kernel: interior + both peer halos
            self.comm.push(ext, x, lay.halo, lay.rows)
            return ext
        ext[lay.halo: lay.halo + lay.rows].copy_(x)
        self.comm.exchange(ext, lay.halo, lay.rows)
        return ext

    def interior(self, ext):
        lay = self.lay
        return ext[lay.halo: lay.halo + lay.rows]

    def gdot(self, pairs):
        return self.comm.allreduce([self.ops.dot(a, b) for a, b in pairs])

    def matvec(self, p):
        """(H^T H / sigma^2 + alpha I) p on the slab: p's halo is the operator's
        reach (2r rows), so each CG iteration exchanges and recomputes 2r rows
        per side, not the denoiser's (70 for PatchWeighted)."""
        ol = self.op_lay
        ext = self.extend(p, "p", ol)
        q = self.ops.normal_matvec(ext, ol.row0, self.H)
        return q[ol.halo: ol.halo + ol.rows].contiguous()

    # -- objective pieces (objective.py:78-121 on slabs)
    def denoise(self, x):
        """f(x) on the slab.  The last result is kept for the same unmodified
        tensor: a cadence cost denoises x_k, and the next fixed-point step
        denoises the same x_k (PatchWeighted is ~60% of a configs[4] step)."""
        c = self._fcache
        if c is not None and c[0] is x and c[1] == x._version:
            return c[2]
        f = self.interior(self.ops.denoise(self.extend(x))).contiguous()
        self._fcache = (x, x._version, f)
        return f

    def cost_terms(self, x):
        f = self.denoise(x)
        ext = self.extend(x)
        fid = self.ops.fidelity(ext, self.yup, self.lay.row0, self.H, self.lay.halo, self.lay.rows)
        vals = [fid, self.ops.dot(x, x), self.ops.dot(x, f)]
        if self.ref is not None:
            vals.append(self.ops.dist2(x, self.ref))
        tot = self.comm.allreduce(vals)
        cost = tot[0] / (2 * self.sigma**2) + self.alpha * 0.5 * (tot[1] - tot[2])
        ps = None
        if self.ref is not None:
            mse = tot[3] / self.N
            ps = math.inf if mse == 0 else (-math.inf if not np.isfinite(mse)
                                            else 10 * math.log10(255.0**2 / mse))
        return cost, ps

    def fp_step(self, x):
        """CG fixed-point step with scipy semantics; returns (x_new, cg_iterations)."""
        ops = self.ops
        f = self.denoise(x)
        b = ops.copy(self.hty)
        ops.axpby(self.alpha, f, 1.0, b)                 # b = hty + alpha f
        xn = ops.copy(x)
        q = self.matvec(xn)
        r = ops.copy(b)
        ops.axpby(-1.0, q, 1.0, r)                       # r = b - A x
        bn2, rho = self.gdot([(b, b), (r, r)])
        bn = math.sqrt(bn2)
        if bn == 0:
            return b, 0
        atol = CG_RTOL * bn
        p = None
        rho_prev = None
        its = 0
        info = CG_MAXITER
        for it in range(CG_MAXITER):
            if math.sqrt(rho) < atol:
                info = 0
                break
            if it > 0:
                ops.axpby(1.0, r, rho / rho_prev, p)      # p = r + beta p
            else:
                p = ops.copy(r)
            q = self.matvec(p)
            (pq,) = self.gdot([(p, q)])
            a = rho / pq
            ops.axpby(a, p, 1.0, xn)
            ops.axpby(-a, q, 1.0, r)
            rho_prev = rho
            (rho,) = self.gdot([(r, r)])
            its += 1
        if info != 0:  # objective.py:114-120
            res = ops.copy(b)
            ops.axpby(-1.0, self.matvec(xn), 1.0, res)
            rn2, bn2b = self.gdot([(res, res), (b, b)])
            if math.sqrt(rn2) > CG_ABORT * math.sqrt(bn2b):
                raise CgNoConvergence(f"CG residual {math.sqrt(rn2):.3e} after {CG_MAXITER} iterations")
        return xn, its

    def gather(self, x, out=None):
        """The full image on every rank (host numpy; a view of ``out``, a
        PinnedHost, when given).  Slabs are gathered where the collective runs
        (device memory under NCCL) and every part goes to the host once."""
        import torch

        H, W = self.H, self.W
        if out is not None and out.shape != (H, W):
            raise ValueError(f"out must be {(H, W)}")
        if self.comm.world == 1:
            if out is None:
                return self.ops.host(x)
            out.t.copy_(x if _io.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x)))
            return out.numpy()
        dist = self.comm.dist
        lays = [SlabLayout(H, W, self.s, self.comm.world, r, 0) for r in range(self.comm.world)]
        maxr = max(l.rows for l in lays)
        buf = torch.zeros((maxr, W), dtype=torch.float64, device=self.comm.device)
        buf[: self.lay.rows].copy_(x if _io.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x)))
        parts = [torch.empty_like(buf) for _ in range(self.comm.world)]
        dist.all_gather(parts, buf, group=self.comm.group)
        dest = out.t if out is not None else torch.from_numpy(np.empty((H, W), dtype=np.float64))
        for l, part in zip(lays, parts):
            dest[l.start: l.stop].copy_(part[: l.rows])
        return dest.numpy()


def _extrapolate(prob, window_list, method, rank_tol):
    """extrapolate_once on a distributed window (extrapolation.py:319-386)."""
    ops = prob.ops
    window = ops.stack(window_list)
    G = np.asarray(prob.comm.allreduce(ops.window_gram(window).ravel().tolist())).reshape(
        len(window_list) - 1, len(window_list) - 1)
    res, xi, need_mgs = ops.decide(G, method, rank_tol)
    if need_mgs:  # exact MGS with distributed inner products (rare)
        res, xi = _mgs_decide(prob, window_list, method, rank_tol)
    if res.converged:
        return "converged", window_list[0], None
    if not res.extrapolated:
        return "skip", window_list[-1], None
    x = ops.combine(window, res.kappa_used, xi)
    k = res.kappa_used
    w = ve.ExtrapolationWeights(method=nat.VE_NAMES[res.method], c=np.array(res.c[: k + 1]),
                                gamma=np.array(res.gamma[: k + 1]),
                                stability_sum=float(res.stability_sum),
                                fallback_from=method if res.fallback else None)
    return "extrapolated", x, w


def _mgs_decide(prob, vs, method, rank_tol):
    ops = prob.ops
    n = len(vs) - 1
    R = np.zeros((n, n))
    Q = []
    rank = n
    r11 = 0.0
    for i in range(n):
        v = ops.copy(vs[i + 1])
        ops.axpby(-1.0, vs[i], 1.0, v)
        for _sweep in range(2):
            for j in range(i):
                (c,) = prob.gdot([(Q[j], v)])
                R[j, i] += c
                ops.axpby(-c, Q[j], 1.0, v)
        (nn,) = prob.gdot([(v, v)])
        rii = math.sqrt(nn)
        R[i, i] = rii
        if i == 0:
            if rii < 1e-300:
                res = nat.VeResultC()
                res.converged = 1
                return res, np.zeros(12)
            r11 = rii
        elif rii < rank_tol * r11:
            rank = i
            break
        ops.axpby(0.0, v, 1.0 / rii, v)
        Q.append(v)
    return ops.decide_r(R, rank, method)


def solve_spatial(prob: SpatialProblem, x0_global, config, reference_trace=True, out=None):
    """run_fixed_point / run_ve_cycling (solvers.py:288-298, 340-385) for one image
    split across ranks.  Returns (x_global on every rank, IterationTrace).
    ``x0_global`` may be a PinnedHost; ``out`` (a PinnedHost) receives the result."""
    method = config.method
    if method not in ("fp", "fp-ve"):
        raise ValueError("spatial solve supports 'fp' and 'fp-ve'")
    if config.ve_method not in METHODS:
        raise ValueError("unknown VE method")
    ops = prob.ops
    x = prob.slab(x0_global)
    trace = IterationTrace()
    every = 1 if prob.N <= DENSE_LOG_LIMIT else 5
    track = method == "fp-ve"
    best_cost, best_x = math.inf, None
    t0 = time.perf_counter()
    k = 0

    def record(xp, xn):
        nonlocal k, best_cost, best_x
        k += 1
        d2, x2 = prob.comm.allreduce([ops.dist2(xn, xp), ops.dot(xp, xp)])
        den = math.sqrt(x2) or 1.0
        sn = math.sqrt(d2) / den
        cost = ps = None
        if k % every == 0:
            cost, ps = prob.cost_terms(xn)
            if track and cost < best_cost:
                best_cost, best_x = cost, ops.copy(xn)
        trace.records.append(TraceRecord(k, cost, ps if prob.ref is not None else None, sn, None,
                                          time.perf_counter() - t0))
        if not (np.isfinite(d2) and np.isfinite(x2)):
            raise NonFiniteIterate(f"iterate diverged at inner step {k}", trace)
        if cost is not None and not np.isfinite(cost):
            raise NonFiniteIterate(f"objective diverged at inner step {k}", trace)
        if sn <= config.tol:
            return "converged"
        if k >= config.max_inner_steps:
            return "budget"
        return None

    if not track:
        while True:
            xn, _ = prob.fp_step(x)
            d = record(x, xn)
            x = xn
            if d is not None:
                break
        return prob.gather(x, out), trace

    c0, _ = prob.cost_terms(x)
    if np.isfinite(c0):
        best_cost, best_x = c0, ops.copy(x)
    clen = config.m + config.kappa + 1
    while True:
        xs = [x]
        conv = False
        for _ in range(clen):
            xn, _ = prob.fp_step(x)
            d = record(x, xn)
            x = xn
            xs.append(x)
            if d == "converged":
                conv = True
                break
            if d == "budget":
                break
        if conv:
            break
        if len(xs) == clen + 1:
            kind, xv, w = _extrapolate(prob, xs[config.m:], config.ve_method, config.rank_tolerance)
            if kind == "converged":
                x = xv
                break
            if kind == "extrapolated":
                (nf,) = prob.comm.allreduce([0.0 if np.isfinite(ops.dot(xv, xv)) else 1.0])
                if nf == 0:
                    x = xv
                    trace.records[-1].gamma_abs_sum = w.stability_sum
                    trace.cycle_weights.append(w)
        if k >= config.max_inner_steps:
            break
    for _ in range(config.stabilization_iters):
        xn, _ = prob.fp_step(x)
        record(x, xn)
        x = xn
    if best_x is not None:
        cf, _ = prob.cost_terms(x)
        if not (np.isfinite(cf) and cf <= best_cost):
            x = best_x
    return prob.gather(x, out), trace
