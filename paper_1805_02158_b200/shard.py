"""Batch sharding across GPUs (BASELINE.json configs[1] and [3]).

One process per GPU; every rank solves a contiguous block of the global batch
with no data-path collective (the images are independent problems).  The
only communication is the optional gather of solutions / per-image status
to rank 0 at the end (``gather=True``), which is result plumbing, not part of
the solve.  SURVEY.md section 8e.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, ragged-tolerant split: the first ``total % world`` ranks take
    one extra image.  Every image belongs to exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def solve_sharded(forward, ys, sigma, alpha, denoiser, x0, config, references=None,
                  gather: bool = False, solve_fn=None):
    """Solve the rank's block of a global batch.

    ``ys`` / ``x0`` / ``references`` hold the GLOBAL batch (host arrays); every
    rank slices its own contiguous block ``[lo:hi)`` out of them.  Returns
    ``(lo, hi, x_local, traces_local, status_local)``; with ``gather=True``
    rank 0 additionally receives ``(x_all, status_all)`` (numpy) as element 5.

    ``solve_fn(forward, ys, sigma, alpha, denoiser, x0, config, refs)`` defaults
    to the device solve; tests inject a CPU stand-in to check the plumbing."""
    d = _dist()
    world = d.get_world_size() if d else 1
    rank = d.get_rank() if d else 0
    total = len(ys)
    lo, hi = shard_bounds(total, world, rank)
    pick = (lambda a: None if a is None else np.asarray(a)[lo:hi])
    if solve_fn is None:
        solve_fn = _device_solve
    x, traces, status = solve_fn(forward, pick(ys), sigma, alpha, denoiser, pick(x0), config,
                                 pick(references))
    x = np.asarray(x)
    status = np.asarray(status, dtype=np.int64)
    out = [lo, hi, x, traces, status]
    if gather:
        if d is None:
            out.append((x, status))
        else:
            import torch

            shape = (hi - lo,) + x.shape[1:]
            counts = [shard_bounds(total, world, r) for r in range(world)]
            maxn = max(h - l for l, h in counts)
            buf = torch.zeros((maxn,) + x.shape[1:], dtype=torch.float64)
            buf[: shape[0]] = torch.from_numpy(x)
            sbuf = torch.zeros(maxn, dtype=torch.int64)
            sbuf[: shape[0]] = torch.from_numpy(status)
            if d.get_backend() == "nccl":
                buf, sbuf = buf.cuda(), sbuf.cuda()
            xs = [torch.empty_like(buf) for _ in range(world)]
            ss = [torch.empty_like(sbuf) for _ in range(world)]
            d.all_gather(xs, buf)
            d.all_gather(ss, sbuf)
            if rank == 0:
                x_all = np.concatenate([xs[r][: counts[r][1] - counts[r][0]].cpu().numpy()
                                        for r in range(world)])
                s_all = np.concatenate([ss[r][: counts[r][1] - counts[r][0]].cpu().numpy()
                                        for r in range(world)])
                out.append((x_all, s_all))
            else:
                out.append(None)
    return tuple(out)


def _device_solve(forward, ys, sigma, alpha, denoiser, x0, config, refs):
    from .batch import RedBatch

    batch = RedBatch(forward, ys, sigma, alpha, denoiser, refs)
    res = batch.solve(x0, config)
    return res.x.cpu().numpy(), [res.trace(b) for b in range(batch.B)], res.status.copy()
