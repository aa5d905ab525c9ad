"""The batch split of configs[1]/[3] (shard.solve_sharded) through its DEVICE
path: two ranks (gloo, sharing the one GPU: their kernels never wait on one
another) each solve their block with libredve_b200 and rank 0 gathers.  The
blocks keep the single-process pairing of images (4 + 4 of 8), so the gathered
solutions equal one single-process batch solve bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SQRT2 = float(np.sqrt(2.0))
B, N, BUDGET = 8, 64, 18


def _inputs():
    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200.synth import voronoi_scene

    op = rv.Blur(rv.make_psf("uniform", 9), (N, N))
    truths = np.stack([voronoi_scene(s, N) for s in range(B)])
    clean = np.asarray(op.apply(truths))
    ys = np.stack([clean[i] + rv.gaussian_noise((N, N), SQRT2, i) for i in range(B)])
    return op, ys


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1805_02158_b200 as rv
        from paper_1805_02158_b200.shard import solve_sharded

        op, ys = _inputs()
        cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=BUDGET)
        out = solve_sharded(op, ys, SQRT2, 0.02, rv.Median3(), ys, cfg, gather=True)
        q.put((rank, out[0], out[1], [t.inner_steps for t in out[3]],
               out[5] if rank == 0 else None))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e), None, None, None))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_device_shards_equal_single_batch():
    import torch.multiprocessing as mp

    import paper_1805_02158_b200 as rv

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for g in got:
        assert not isinstance(g[1], str), g[1]
    assert (got[0][1], got[0][2], got[1][1], got[1][2]) == (0, 4, 4, 8)
    assert got[0][3] == [BUDGET] * 4 and got[1][3] == [BUDGET] * 4
    x_all, s_all = got[0][4]
    op, ys = _inputs()
    cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=BUDGET)
    X, _ = rv.solve_batch(rv.RedBatch(op, ys, SQRT2, 0.02, rv.Median3()), ys, cfg)
    np.testing.assert_array_equal(x_all, X.cpu().numpy())
    assert (s_all == 0).all()
