"""Multi-process (world_size 2, gloo, CPU) checks of the batch-sharding plumbing.

The per-rank solver is the CPU oracle injected through ``solve_fn`` (the GPU
solve is covered by the -m gpu tests); what is tested here is the split, the
independence of the shards and the gather to rank 0."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_02158_b200.shard import shard_bounds, solve_sharded

SQRT2 = float(np.sqrt(2.0))


def test_shard_bounds_cover_and_balance():
    for total in (0, 1, 5, 64, 65, 512):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _oracle_solve(forward, ys, sigma, alpha, denoiser, x0, config, refs):
    from oracle import extras
    from oracle import redve_ref as R

    n = ys.shape[1]
    op = R.CirculantBlur(R.psf_taps("uniform", 9), (n, n))
    xs, traces, status = [], [], []
    for b in range(len(ys)):
        step, cost = R.red_problem(R.Red(op, ys[b], sigma, alpha, extras.median3))
        x, tr = R.run_cycling(step, x0[b], config["budget"], "mpe", objective=cost)
        xs.append(x.reshape(n, n))
        traces.append(tr)
        status.append(0)
    return np.stack(xs), traces, np.array(status)


def _inputs(total=5, n=32):
    from oracle import redve_ref as R
    from paper_1805_02158_b200.synth import voronoi_scene

    op = R.CirculantBlur(R.psf_taps("uniform", 9), (n, n))
    truths = np.stack([voronoi_scene(s, n) for s in range(total)])
    ys = np.stack([R.measure(truths[i], op, SQRT2, i) for i in range(total)])
    return ys


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ys = _inputs()
        out = solve_sharded(None, ys, SQRT2, 0.02, None, ys, {"budget": 12}, gather=True,
                            solve_fn=_oracle_solve)
        lo, hi = out[0], out[1]
        q.put((rank, lo, hi, out[5] if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gather_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    assert got[0][1:3] == (0, 3) and got[1][1:3] == (3, 5)
    x_all, s_all = got[0][3]
    ys = _inputs()
    ref, _, _ = _oracle_solve(None, ys, SQRT2, 0.02, None, ys, {"budget": 12}, None)
    np.testing.assert_array_equal(x_all, ref)  # shards are independent: bit-identical
    assert (s_all == 0).all()
