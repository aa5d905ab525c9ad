"""solve_stream (copies of the neighbouring batches under a batch's kernels)
returns exactly what serial RedBatch + solve_batch calls return."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _batches(n, B, nb):
    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200.synth import voronoi_scene

    op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
    out = []
    for k in range(nb):
        truths = np.stack([voronoi_scene(100 * k + s, n) for s in range(B)])
        clean = np.asarray(op.apply(truths))
        out.append(np.stack([clean[i] + rv.gaussian_noise((n, n), float(np.sqrt(2)), 7 * k + i)
                             for i in range(B)]))
    return op, out


@pytest.mark.parametrize("pinned", [False, True])
def test_solve_stream_equals_serial(pinned):
    import paper_1805_02158_b200 as rv

    n, B, nb = 64, 4, 5
    op, ys = _batches(n, B, nb)
    sig = float(np.sqrt(2))
    cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", m=0, kappa=5, max_inner_steps=36)
    serial = []
    for y in ys:
        X, trs = rv.solve_batch(rv.RedBatch(op, y, sig, 0.02, rv.Median3()), y, cfg)
        serial.append((X.cpu().numpy(), trs))
    got = []
    import torch

    src = [torch.from_numpy(y).pin_memory() for y in ys] if pinned else ys
    for xh, trs in rv.solve_stream(op, iter(src), sig, 0.02, rv.Median3(), cfg):
        got.append((xh.numpy().copy(), trs))  # the pinned slot is reused later
    assert len(got) == nb
    for (xs, ts), (xp, tp) in zip(serial, got):
        np.testing.assert_array_equal(xs, xp)
        for a, b in zip(ts, tp):
            assert a.inner_steps == b.inner_steps
            np.testing.assert_array_equal([r.step_norm for r in a.records],
                                          [r.step_norm for r in b.records])


def test_solve_stream_x0_and_empty():
    import paper_1805_02158_b200 as rv

    n, B = 48, 2
    op, ys = _batches(n, B, 2)
    sig = float(np.sqrt(2))
    cfg = rv.SolveConfig(method="fp", max_inner_steps=12)
    x0 = [np.zeros_like(y) for y in ys]
    res = [(xh.numpy().copy(), trs)
           for xh, trs in rv.solve_stream(op, zip(ys, x0), sig, 0.02, rv.GaussianFilter(), cfg)]
    for (xh, trs), y, z in zip(res, ys, x0):
        X, _ = rv.solve_batch(rv.RedBatch(op, y, sig, 0.02, rv.GaussianFilter()), z, cfg)
        np.testing.assert_array_equal(X.cpu().numpy(), xh)
    assert list(rv.solve_stream(op, iter([]), sig, 0.02, rv.Median3(), cfg)) == []


@pytest.mark.parametrize("route", ["fourier-median", "spectral-gaussian", "cg-sr"])
def test_set_measurements_equals_fresh_problem(route):
    """RedBatch.set_measurements == a fresh RedBatch on the new measurements, on
    every route, with the solve graph captured once."""
    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200.synth import voronoi_scene

    if route == "cg-sr":
        n, B = 48, 2
        op = rv.BlurDownsample(rv.make_psf("gaussian", 7, 1.6), 3, (n, n))
        den, sig = rv.GaussianFilter(), 5.0
        cfg = rv.SolveConfig(method="fp-ve", ve_method="rre", m=0, kappa=3, max_inner_steps=10)
    else:
        n, B = 64, 3
        op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
        den = rv.Median3() if route == "fourier-median" else rv.GaussianFilter()
        sig = float(np.sqrt(2))
        cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", m=0, kappa=5, max_inner_steps=30)
    sets = []
    for k in range(3):
        truths = np.stack([voronoi_scene(50 * k + s, n) for s in range(B)])
        ys = np.stack([rv.degrade(truths[i], op, sig, 11 * k + i) for i in range(B)])
        x0 = np.asarray(op.adjoint(ys)) if route == "cg-sr" else ys
        sets.append((truths, ys, x0))
    fresh = []  # first: the executable graph of this topology is handed from problem to problem
    for truths, ys, x0 in sets:
        Xf, tf = rv.solve_batch(rv.RedBatch(op, ys, sig, 0.02, den, truths), x0, cfg)
        fresh.append((Xf.cpu().numpy(), tf))
    kept = rv.RedBatch(op, sets[0][1], sig, 0.02, den, sets[0][0])
    for k, (truths, ys, x0) in enumerate(sets):
        if k:
            kept.set_measurements(ys, truths)
        Xk, tk = rv.solve_batch(kept, x0, cfg)
        Xf, tf = fresh[k]
        np.testing.assert_array_equal(Xk.cpu().numpy(), Xf)
        for a, b in zip(tk, tf):
            assert a.inner_steps == b.inner_steps
            np.testing.assert_array_equal(a.costs(), b.costs())
            np.testing.assert_array_equal([r.psnr for r in a.records], [r.psnr for r in b.records])
    if route != "cg-sr":
        assert kept.graph_captures == 1
    with pytest.raises(ValueError):
        kept.set_measurements(sets[0][1])  # created with references
    with pytest.raises(rv.ShapeMismatch):
        kept.set_measurements(sets[0][1][:1], sets[0][0][:1])
