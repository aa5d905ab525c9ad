"""GPU parity of the spatially partitioned SR solve (configs[4]):
the native slab primitives against the CPU stand-in / numpy, and the whole
distributed driver over libredve_b200 against the single-domain oracle, on one
rank and on two ranks sharing the GPU (gloo host collectives; the ranks'
kernels never wait on one another)."""

import os

import numpy as np
import pytest
import torch.distributed as dist

from test_spatial_gloo import ALPHA, FACTOR, SIGMA, _Fwd, _free_port, _oracle, _setup

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def pair():
    import torch

    from oracle import extras
    from paper_1805_02158_b200 import Median3
    from paper_1805_02158_b200.spatial import NativeSlabOps
    from spatial_cpu_ops import CpuSlabOps

    taps, op, truth, y, den, reach, x0 = _setup(60, 47, "median")
    fwd = _Fwd(taps, FACTOR, (60, 47))
    nat = NativeSlabOps(fwd, SIGMA, ALPHA, Median3())
    cpu = CpuSlabOps(taps, FACTOR, SIGMA, ALPHA, extras.median3)
    return nat, cpu, torch


def test_reductions_and_update(pair):
    nat, cpu, torch = pair
    g = np.random.default_rng(1)
    a, b = g.standard_normal((37, 53)) * 50, g.standard_normal((37, 53)) * 50
    ta, tb = nat.tensor(a), nat.tensor(b)
    assert abs(nat.dot(ta, tb) - float(np.vdot(a, b))) <= 1e-12 * abs(float(np.vdot(a, a)))
    assert nat.dist2(ta, tb) == pytest.approx(float(((a - b) ** 2).sum()), rel=1e-13)
    assert nat.dot(nat.zeros((0,)), nat.zeros((0,))) == 0.0
    nat.axpby(0.5, ta, -2.0, tb)
    np.testing.assert_allclose(nat.host(tb), 0.5 * a - 2.0 * b, rtol=1e-15, atol=1e-12)


@pytest.mark.parametrize("row0,Hg", [(0, 60), (7, 60), (58, 60), (13, 8192)])
def test_normal_matvec_and_fidelity_on_global_lattice(pair, row0, Hg):
    nat, cpu, torch = pair
    g = np.random.default_rng(row0)
    w = g.uniform(0, 255, (40, 47))
    got = nat.host(nat.normal_matvec(nat.tensor(w), row0, Hg))
    want = cpu.host(cpu.normal_matvec(cpu.tensor(w), row0, Hg))
    assert rel(got, want) <= 1e-12
    yup = cpu._mask(w.shape, row0, Hg) * g.uniform(0, 255, w.shape)
    f_nat = nat.fidelity(nat.tensor(w), nat.tensor(yup), row0, Hg, 6, 28)
    f_cpu = cpu.fidelity(cpu.tensor(w), cpu.tensor(yup), row0, Hg, 6, 28)
    assert f_nat == pytest.approx(f_cpu, rel=1e-12)
    c_nat = nat.host(nat.correlate(nat.tensor(yup), 0.04))
    c_cpu = cpu.host(cpu.correlate(cpu.tensor(yup), 0.04))
    assert rel(c_nat, c_cpu) <= 1e-12


@pytest.mark.parametrize("method", ["mpe", "rre", "svdmpe"])
def test_window_gram_decide_combine(pair, method):
    from oracle import redve_ref as R

    nat, cpu, torch = pair
    g = np.random.default_rng(5)
    rows = 7
    base = g.standard_normal((33, 29))
    win = np.stack([base * 0.7**k + g.standard_normal(base.shape) * 1e-2 for k in range(rows)])
    G = nat.window_gram(nat.tensor(win))
    Gc = cpu.window_gram(cpu.tensor(win))
    assert rel(G, Gc) <= 1e-12
    res, xi, need = nat.decide(G, method, 1e-12)
    assert not need and res.extrapolated
    out = nat.host(nat.combine(nat.tensor(win), res.kappa_used, xi))
    ref = R.extrapolate(win.reshape(rows, -1), method)
    assert res.kappa_used == ref["kappa_used"]
    np.testing.assert_allclose(np.array(res.gamma[: res.kappa_used + 1]), ref["gamma"], rtol=1e-7)
    assert rel(out.ravel(), ref["vector"]) <= 1e-10


def _native_spatial(H, W, method, budget, ve_method, den_name="median", comm=None, pinned=False):
    from paper_1805_02158_b200 import Median3, PatchWeighted
    from paper_1805_02158_b200.solvers import SolveConfig
    from paper_1805_02158_b200.spatial import (PeerComm, PinnedHost, SpatialProblem, TorchComm,
                                               solve_spatial)

    if comm == "peer":                     # built inside the rank process
        comm = PeerComm(device="cpu")

    taps, op, truth, y, _, _, x0 = _setup(H, W, "median")
    den = Median3() if den_name == "median" else PatchWeighted(1, 1, 110.0, 3)
    out = None
    if pinned:  # page-locked host images in, result into a caller-owned pinned buffer
        y, x0, truth, out = PinnedHost(y), PinnedHost(x0), PinnedHost(truth), PinnedHost(shape=(H, W))
    prob = SpatialProblem(_Fwd(taps, FACTOR, (H, W)), y, SIGMA, ALPHA, den,
                          comm=comm or TorchComm(), reference=truth)
    cfg = SolveConfig(method=method, ve_method=ve_method, max_inner_steps=budget)
    x, tr = solve_spatial(prob, x0, cfg, out=out)
    if pinned:
        assert np.shares_memory(x, out.numpy()) and out.t.is_pinned()
        x = x.copy()
    return (x, np.array([r.step_norm for r in tr.records]),
            np.array([np.nan if r.cost is None else r.cost for r in tr.records]),
            np.array([np.nan if r.psnr is None else r.psnr for r in tr.records]))


def _check(got, H, W, method, budget, ve_method, den_name="median"):
    x, sn, cost, ps = got
    if den_name == "median":
        xr, tr = _oracle(H, W, "median", method, budget, ve_method)
    else:
        from oracle import redve_ref as R

        taps, op, truth, y, _, _, x0 = _setup(H, W, "median")
        dn = lambda v: R.patch_weighted(v, 1, 1, 110.0, 3)
        step, costf = R.red_problem(R.Red(op, y, SIGMA, ALPHA, dn))
        xr, tr = R.run_cycling(step, x0, budget, ve_method, objective=costf,
                               reference=truth.ravel())
        xr = xr.reshape(H, W)
    a = tr.as_arrays()
    assert len(sn) == len(a["step_norm"])           # same iteration count
    assert rel(x, xr) <= 1e-5                        # north_star bar
    np.testing.assert_allclose(sn, a["step_norm"], rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(cost, a["cost"], rtol=1e-7)
    np.testing.assert_allclose(ps, a["psnr"], atol=0.01)


@pytest.mark.parametrize("method,ve_method", [("fp-ve", "rre"), ("fp-ve", "mpe"), ("fp", "rre")])
def test_single_rank_native_solve(method, ve_method):
    _check(_native_spatial(96, 90, method, 14, ve_method), 96, 90, method, 14, ve_method)


def test_single_rank_native_patch_weighted():
    _check(_native_spatial(66, 60, "fp-ve", 14, "rre", "pw"), 66, 60, "fp-ve", 14, "rre", "pw")


def _worker(rank, world, port, q, args):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        q.put((rank, _native_spatial(*args)))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_native_solve():
    import torch.multiprocessing as mp

    H, W, budget = 96, 90, 14
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (H, W, "fp-ve", budget, "rre")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, args)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(out[r], str), out[r]
    for k in range(4):
        np.testing.assert_array_equal(out[0][k], out[1][k])
    _check(out[0], H, W, "fp-ve", budget, "rre")


def test_pinned_host_images_equal_numpy_images():
    """PinnedHost inputs / output buffer: the same solve, bit for bit."""
    got = _native_spatial(96, 90, "fp-ve", 14, "rre", pinned=True)
    ref = _native_spatial(96, 90, "fp-ve", 14, "rre")
    for k in range(4):
        np.testing.assert_array_equal(got[k], ref[k])


# ---- peer-memory halo exchange (PeerComm / redve_halo_push) ----------------
def test_single_rank_peer_push_solve():
    from paper_1805_02158_b200.spatial import PeerComm

    got = _native_spatial(96, 90, "fp-ve", 14, "rre", comm=PeerComm())
    ref = _native_spatial(96, 90, "fp-ve", 14, "rre")
    for k in range(4):
        np.testing.assert_array_equal(got[k], ref[k])  # same halos -> same bits


def _push_worker(rank, world, port, q, args):
    """Every rank pushes a slab whose values encode (global row, column); the
    extended buffers must then hold the ring's rows exactly."""
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1805_02158_b200.spatial import PeerComm, SlabLayout

        H, W, factor, halo = args
        comm = PeerComm(device="cpu")
        lay = SlabLayout(H, W, factor, world, rank, halo)
        g = torch.arange(H, dtype=torch.float64, device="cuda")[:, None] * 1000 + \
            torch.arange(W, dtype=torch.float64, device="cuda")[None, :]
        ext = torch.full((lay.Hext, W), -1.0, dtype=torch.float64, device="cuda")
        bad = 0
        for rnd in range(3):                       # repeated pushes reuse the mappings
            x = g[lay.start: lay.stop] + rnd
            comm.push(ext, x, halo, lay.rows)
            want = g[torch.tensor(lay.ext_rows(), device="cuda")] + rnd
            bad += int((ext != want).sum().item())
        q.put((rank, (bad, lay.rows, hasattr(ext, "_redve_peer"))))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,W,halo", [(2, 99, 47, 4), (3, 99, 64, 3), (2, 60, 10, 30)])
def test_peer_push_ring(world, H, W, halo):
    """Ragged slabs (99 rows / factor 3 does not split evenly), odd and even
    widths (scalar and 16-byte paths), and a halo as thick as the slab."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_push_worker, args=(r, world, port, q, (H, W, 3, halo)))
             for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
        assert out[r][0] == 0 and out[r][2]
    if (world, H) == (2, 99):
        assert len({out[r][1] for r in range(world)}) > 1  # really ragged (51 / 48)


def test_two_ranks_peer_push_solve():
    """The distributed solve with peer-memory halos equals the send/recv one."""
    import torch.multiprocessing as mp

    H, W, budget = 96, 90, 14
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (H, W, "fp-ve", budget, "rre", "median", "peer")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, args)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(out[r], str), out[r]
    for k in range(4):
        np.testing.assert_array_equal(out[0][k], out[1][k])
    _check(out[0], H, W, "fp-ve", budget, "rre")
