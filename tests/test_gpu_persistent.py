"""The persistent TMA-fed column pass (k_col_p in csrc/fourier.cu) against the
one-shot k_col (REDVE_PERSISTENT=0) on the same inputs: both do the same
arithmetic in the same order (the spectral scaling is explicitly rounded, so
no contraction differs), so iterates and traces agree bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SQRT2 = float(np.sqrt(2.0))


@pytest.fixture(scope="module")
def rv():
    import paper_1805_02158_b200 as rv

    return rv


def _problem(rv, B, n, den):
    from paper_1805_02158_b200.synth import voronoi_scene

    op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
    truths = np.stack([voronoi_scene(s, n) for s in range(B)])
    clean = np.asarray(op.apply(truths))
    ys = np.stack([clean[i] + rv.gaussian_noise((n, n), SQRT2, i) for i in range(B)])
    dn = {"median": rv.Median3, "gauss": rv.GaussianFilter, "fb": lambda: rv.FilterBank(0)}[den]()
    return op, ys, dn, truths


def _run(rv, monkeypatch, flag, B, n, den, cfg):
    monkeypatch.setenv("REDVE_PERSISTENT", flag)
    monkeypatch.setenv("REDVE_SPECTRAL", "0")  # keep linear denoisers on the Fourier kernels
    op, ys, dn, truths = _problem(rv, B, n, den)
    batch = rv.RedBatch(op, ys, SQRT2, 0.02, dn, truths)
    res = batch.solve(ys, cfg)
    return res.x.cpu().numpy(), res


@pytest.mark.parametrize("B,n,den", [(5, 128, "median"), (6, 256, "gauss"), (3, 512, "fb"),
                                     (64, 256, "median")])
@pytest.mark.parametrize("method,ve", [("fp", "mpe"), ("fp-ve", "rre")])
def test_persistent_equals_one_shot(rv, monkeypatch, B, n, den, method, ve):
    cfg = rv.SolveConfig(method=method, ve_method=ve, max_inner_steps=30)
    x1, r1 = _run(rv, monkeypatch, "1", B, n, den, cfg)
    x0, r0 = _run(rv, monkeypatch, "0", B, n, den, cfg)
    np.testing.assert_array_equal(x1, x0)
    np.testing.assert_array_equal(r1.n_records, r0.n_records)
    np.testing.assert_array_equal(r1.step_norm, r0.step_norm)
    np.testing.assert_array_equal(r1.cost, r0.cost)


def test_persistent_skips_finished_images(rv, monkeypatch):
    """tol > 0: images stop at different steps, so later passes skip the tiles of
    finished pairs."""
    cfg = rv.SolveConfig(method="fp", max_inner_steps=60, tol=2e-3)
    x1, r1 = _run(rv, monkeypatch, "1", 7, 256, "median", cfg)
    x0, r0 = _run(rv, monkeypatch, "0", 7, 256, "median", cfg)
    assert len(set(r0.n_records.tolist())) > 1, "images should stop at different steps"
    np.testing.assert_array_equal(r1.n_records, r0.n_records)
    np.testing.assert_array_equal(x1, x0)
