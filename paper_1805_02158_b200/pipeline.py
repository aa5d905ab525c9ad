"""Pipelined batch solves: host copies of neighbouring batches ride under the kernels.

A solve of one batch is [H2D of the measurements, problem setup, the device
schedule, D2H of the solutions].  Run back to back, the copies leave the SMs
idle (configs[1]: ~1.4 ms of a 21 ms step).  ``solve_stream`` uploads batch
i+1 and downloads batch i-1 on a copy stream while batch i's schedule runs on
the compute stream (one solve at a time: two schedules sharing the SMs were
measured slower than one after the other), and the batches share one
``RedBatch`` whose measurements are replaced (``set_measurements``), so the
solve schedule is captured once.  Every batch computes what an independent
``RedBatch`` + ``solve_batch`` computes (objective.py:44-74,
solvers.py:388-399), bit for bit; results come back in submission order, one
batch behind the solves.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _io
from .batch import RedBatch, solve_batch

__all__ = ["solve_stream"]


def solve_stream(forward, batches, sigma, alpha, denoiser, config, references=None):
    """Solve a sequence of batches; yields ``(x_host, traces)`` per batch, in order.

    ``batches`` yields ``ys`` or ``(ys, x0)`` (numpy arrays or host tensors,
    pinned ones are uploaded without a staging copy; ``x0=None`` starts from the
    measurements, cli.py:362-363).  ``x_host`` is a pinned host tensor owned by
    the pipeline: it stays valid until the next result has been taken from the
    generator.  Per-image failures raise as in ``solve_batch``."""
    torch = _io.torch_mod()
    device = torch.cuda.current_device()
    main = torch.cuda.current_stream(device)
    copy = torch.cuda.Stream(device=device)
    stage = {}  # pinned staging buffers for unpinned inputs, by (tag, parity)

    def to_pinned(a, tag, parity):
        if a is None:
            return None
        if isinstance(a, torch.Tensor):
            if a.is_cuda or a.is_pinned():
                return a
            src = a.to(torch.float64)
        else:
            src = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
        buf = stage.get((tag, parity))
        if buf is None or buf.shape != src.shape:
            buf = stage[(tag, parity)] = torch.empty(src.shape, dtype=torch.float64).pin_memory()
        buf.copy_(src)
        return buf

    def upload(item, parity):
        """Runs on the helper thread: stage, then H2D on the copy stream."""
        ys, x0 = item if isinstance(item, tuple) else (item, None)
        with torch.cuda.device(device), torch.cuda.stream(copy):
            out = []
            for tag, a in (("y", ys), ("x0", x0)):
                h = to_pinned(a, tag, parity)
                if h is None:
                    out.append(None)
                    continue
                d = h if h.is_cuda else h.to("cuda", dtype=torch.float64, non_blocking=True)
                d.record_stream(main)
                out.append(d)
            ev = torch.cuda.Event()
            ev.record(copy)
        return out[0], out[1], ev

    class _Now:  # an upload issued inline (future-like)
        def __init__(self, value):
            self.value = value

        def result(self):
            return self.value

    def staged(item):
        """Needs a host-side staging copy (unpinned input): worth a helper thread."""
        parts = item if isinstance(item, tuple) else (item,)
        return any(a is not None and not (isinstance(a, torch.Tensor) and (a.is_cuda or a.is_pinned()))
                   for a in parts)

    slots = [None, None]
    batch = None
    done = None  # (slot tensor, traces, event) of the previous batch
    it = iter(batches)
    with ThreadPoolExecutor(max_workers=1, thread_name_prefix="redve-upload") as pool:
        def start(item, parity):
            # pinned / device inputs: the upload is one asynchronous copy, issued
            # inline; unpinned ones are staged on the helper thread meanwhile
            return pool.submit(upload, item, parity) if staged(item) else _Now(upload(item, parity))

        try:
            nxt = start(next(it), 0)
        except StopIteration:
            return
        i = 0
        while nxt is not None:
            y_dev, x0_dev, ev = nxt.result()
            try:
                nxt = start(next(it), (i + 1) & 1)
            except StopIteration:
                nxt = None
            main.wait_event(ev)
            # one problem for the whole stream: new measurements into the same
            # device buffers, the solve schedule captured once and replayed
            if batch is None or tuple(batch.y.shape) != tuple(y_dev.shape):
                batch = RedBatch(forward, y_dev, sigma, alpha, denoiser, references)
            else:
                batch.set_measurements(y_dev, references)
            X, traces = solve_batch(batch, y_dev if x0_dev is None else x0_dev, config)
            s = i & 1
            if slots[s] is None or slots[s].shape != X.shape:
                slots[s] = torch.empty(X.shape, dtype=X.dtype).pin_memory()
            copy.wait_stream(main)
            with torch.cuda.stream(copy):
                slots[s].copy_(X, non_blocking=True)
                dev = torch.cuda.Event()
                dev.record(copy)
            X.record_stream(copy)
            del X
            if done is not None:
                done[2].synchronize()
                yield done[0], done[1]
            done = (slots[s], traces, dev)
            i += 1
        if done is not None:
            done[2].synchronize()
            yield done[0], done[1]
