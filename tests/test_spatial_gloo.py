"""Spatially partitioned SR solve (configs[4]): the distributed
driver over row slabs, halo exchange and allreduced inner products, run with
world_size 1 and 2 (gloo, CPU) against the single-domain oracle solve.

The slab algebra here is the CPU stand-in (tests/spatial_cpu_ops.py, built on
the oracle); the native slab primitives are covered by test_gpu_spatial in
test_gpu_parity.py.  What is tested: partition and halo bookkeeping, the
periodic ring, the global measurement lattice on slabs that do not start on a
multiple of the factor, and the driver's decisions being rank-identical."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_02158_b200.spatial import SlabLayout

SIGMA, ALPHA, FACTOR = 5.0, 0.05, 3


def test_slab_layout_covers_and_respects_phase():
    for H in (50, 51, 96, 8192):
        for world in (1, 2, 3, 8):
            if -(-H // FACTOR) < world:
                continue
            lays = [SlabLayout(H, 7, FACTOR, world, r, 0) for r in range(world)]
            assert lays[0].start == 0 and lays[-1].stop == H
            for a, b in zip(lays, lays[1:]):
                assert a.stop == b.start
                assert b.start % FACTOR == 0
    lay = SlabLayout(50, 7, FACTOR, 2, 1, 6)
    assert lay.row0 == (lay.start - 6) % 50 and lay.Hext == lay.rows + 12
    with pytest.raises(ValueError):
        SlabLayout(12, 7, FACTOR, 2, 0, 7)


class _Fwd:
    def __init__(self, taps, factor, shape):
        from paper_1805_02158_b200.imaging import Psf

        self.psf = Psf(taps.shape[0], taps)
        self.factor = factor
        self.in_shape = shape


def _setup(H, W, denoiser_name):
    from oracle import extras
    from oracle import redve_ref as R

    taps = R.psf_taps("gaussian", 7, 1.6)
    op = R.BlurDecimate(taps, FACTOR, (H, W))
    truth = R.scene(H, W)
    y = R.measure(truth, op, SIGMA, 3)
    den, reach = {"median": (extras.median3, 1), "gauss": (R.gaussian_filter, 2)}[denoiser_name]
    x0 = np.kron(y, np.ones((FACTOR, FACTOR)))[:H, :W]
    return taps, op, truth, y, den, reach, x0


def _oracle(H, W, denoiser_name, method, budget, ve_method="rre"):
    from oracle import redve_ref as R

    taps, op, truth, y, den, reach, x0 = _setup(H, W, denoiser_name)
    step, cost = R.red_problem(R.Red(op, y, SIGMA, ALPHA, den))
    if method == "fp":
        x, tr = R.run_fp(step, x0, budget, objective=cost, reference=truth.ravel())
    else:
        x, tr = R.run_cycling(step, x0, budget, ve_method, objective=cost, reference=truth.ravel())
    return x.reshape(H, W), tr


def _spatial(H, W, denoiser_name, method, budget, ve_method="rre"):
    from paper_1805_02158_b200.solvers import SolveConfig
    from paper_1805_02158_b200.spatial import SpatialProblem, TorchComm, solve_spatial
    from spatial_cpu_ops import CpuSlabOps

    taps, op, truth, y, den, reach, x0 = _setup(H, W, denoiser_name)
    ops = CpuSlabOps(taps, FACTOR, SIGMA, ALPHA, den)
    prob = SpatialProblem(_Fwd(taps, FACTOR, (H, W)), y, SIGMA, ALPHA, None, comm=TorchComm(),
                          ops=ops, reference=truth, reach=reach)
    cfg = SolveConfig(method=method, ve_method=ve_method, max_inner_steps=budget)
    x, tr = solve_spatial(prob, x0, cfg)
    sn = [r.step_norm for r in tr.records]
    cost = [np.nan if r.cost is None else r.cost for r in tr.records]
    ps = [np.nan if r.psnr is None else r.psnr for r in tr.records]
    gam = [np.nan if r.gamma_abs_sum is None else r.gamma_abs_sum for r in tr.records]
    return x, np.array(sn), np.array(cost), np.array(ps), np.array(gam)


def _compare(got, H, W, den, method, budget, ve_method="rre"):
    x, sn, cost, ps, gam = got
    xr, tr = _oracle(H, W, den, method, budget, ve_method)
    a = tr.as_arrays()
    assert len(sn) == len(a["step_norm"])
    assert np.linalg.norm(x - xr) <= 1e-9 * np.linalg.norm(xr)
    np.testing.assert_allclose(sn, a["step_norm"], rtol=1e-6, atol=1e-14)
    np.testing.assert_allclose(cost, a["cost"], rtol=1e-9)
    np.testing.assert_allclose(ps, a["psnr"], atol=1e-6)
    np.testing.assert_allclose(gam, a["gamma_abs_sum"], rtol=1e-6)


@pytest.mark.parametrize("method,den", [("fp-ve", "median"), ("fp", "gauss")])
def test_single_rank_matches_oracle(method, den):
    _compare(_spatial(50, 47, den, method, 14), 50, 47, den, method, 14)


def _worker(rank, world, port, q, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _spatial(*args)))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_world(world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    return out


@pytest.mark.parametrize("method,den,ve_method", [("fp-ve", "median", "rre"),
                                                  ("fp-ve", "median", "mpe"),
                                                  ("fp", "gauss", "rre")])
def test_two_ranks_match_oracle(method, den, ve_method):
    H, W, budget = 50, 47, 14
    out = _run_world(2, (H, W, den, method, budget, ve_method))
    # every rank holds the same gathered image and the same trace
    for k in range(5):
        np.testing.assert_array_equal(out[0][k], out[1][k])
    _compare(out[0], H, W, den, method, budget, ve_method)


def test_three_ranks_ragged_slabs_match_oracle():
    """Three slabs of unequal height (18, 18, 14 rows), the last not ending on
    a measurement row, the periodic ring closing over three neighbours."""
    H, W, budget = 50, 47, 14
    out = _run_world(3, (H, W, "median", "fp-ve", budget, "rre"))
    for r in (1, 2):
        for k in range(5):
            np.testing.assert_array_equal(out[0][k], out[r][k])
    _compare(out[0], H, W, "median", "fp-ve", budget, "rre")
