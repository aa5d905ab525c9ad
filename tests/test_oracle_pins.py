"""Pin the CPU oracle (oracle/redve_ref.py) to the reference before trusting it.

Fixtures come from the unmodified reference (tests/golden/make_golden.py) and
from its byte-reproducible demo traces (pkg/demos/out/deblur_*.csv).  CPU only.
"""

import numpy as np
import pytest
from scipy import ndimage

from oracle import extras
from oracle import redve_ref as R

SQRT2 = float(np.sqrt(2.0))


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _trace_close(tr, g, prefix, rtol=1e-10):
    t = tr.as_arrays()
    assert np.array_equal(t["iter"], g[f"{prefix}/iter"])
    for key in ("cost", "psnr", "gamma_abs_sum"):
        a, b = t[key], g[f"{prefix}/{key}"]
        assert np.array_equal(np.isnan(a), np.isnan(b)), key
        m = ~np.isnan(b)
        np.testing.assert_allclose(a[m], b[m], rtol=rtol, atol=0, err_msg=key)
    sn_a, sn_b = t["step_norm"], g[f"{prefix}/step_norm"]
    m = sn_b > 1e-12  # below that the step norm is FFT rounding noise
    np.testing.assert_allclose(sn_a[m], sn_b[m], rtol=1e-6)
    assert len(tr.cycles) == int(g[f"{prefix}/n_cycles"])


@pytest.fixture(scope="module")
def runs(golden):
    g = golden("demo64.npz")
    truth, y = g["truth"], g["y"]
    op = R.CirculantBlur(R.psf_taps("uniform", 9), truth.shape)
    np.testing.assert_array_equal(R.measure(truth, op, SQRT2, 0), y)  # bit-identical noise
    red = R.Red(op, y, SQRT2, 0.02, R.gaussian_filter)
    step, cost = R.red_problem(red)
    fp = R.run_fp(step, y, 120, objective=cost, reference=truth.ravel())
    mpe = R.run_cycling(step, y, 120, "mpe", objective=cost, reference=truth.ravel())
    return g, fp, mpe


class TestDemoKAT:
    """pkg/demos/out/deblur_{fp,fp-mpe}.csv known-answer traces (64^2, budget 120)."""

    @pytest.mark.parametrize("name", ["fp", "fp-mpe"])
    def test_trace_matches_csv(self, runs, name):
        g, fp, mpe = runs
        tr = (fp if name == "fp" else mpe)[1].as_arrays()
        np.testing.assert_array_equal(tr["iter"], g[f"{name}/iter"])
        np.testing.assert_allclose(tr["cost"], g[f"{name}/cost"], rtol=1e-12)
        np.testing.assert_allclose(tr["psnr"], g[f"{name}/psnr"], rtol=1e-12)
        b = g[f"{name}/gamma_abs_sum"]
        assert np.array_equal(np.isnan(tr["gamma_abs_sum"]), np.isnan(b))
        m = g[f"{name}/step_norm"] > 1e-12
        np.testing.assert_allclose(tr["step_norm"][m], g[f"{name}/step_norm"][m], rtol=1e-9)

    def test_crossing_at_31(self, runs):
        g, fp, mpe = runs
        target = fp[1].cost[-1]
        assert abs(target - 2787.1615224101) < 1e-6
        assert mpe[1].first_iter_at_cost(target) == 31


class TestVeWindows:
    CASES = ["random0", "random1", "random2", "random3", "random4", "random5", "linear_k3",
             "linear_k5_rankdef", "rank1", "stationary", "mpe_degenerate", "oscillating", "decay_k5"]

    @pytest.mark.parametrize("case", CASES)
    @pytest.mark.parametrize("method", ["mpe", "rre", "svdmpe"])
    def test_extrapolate_matches_reference(self, golden, case, method):
        g = golden("ve_windows.npz")
        rows = g[f"{case}/rows"]
        res = R.extrapolate(rows, method)
        key = f"{case}/{method}"
        flags = g[f"{key}/flags"]
        assert int(res["converged"]) == flags[0]
        assert int(res["extrapolated"]) == flags[1]
        assert res["kappa_used"] == flags[2]
        if flags[3] >= 0:
            assert int(res["fallback_from"] is not None) == flags[3]
            np.testing.assert_allclose(res["gamma"], g[f"{key}/gamma"], rtol=1e-12, atol=1e-14)
            assert abs(res["stability_sum"] - float(g[f"{key}/stability"])) <= 1e-12 * float(
                g[f"{key}/stability"])
        np.testing.assert_allclose(res["vector"], g[f"{key}/vector"], rtol=1e-12, atol=1e-12)


class TestOperatorsDenoisers:
    def test_all(self, golden):
        g = golden("operators.npz")
        i = 0
        while f"x{i}" in g:
            x = g[f"x{i}"]
            shp = x.shape
            np.testing.assert_allclose(R.gaussian_filter(x), g[f"gauss{i}"], rtol=1e-14, atol=1e-12)
            if min(shp) >= 5:
                np.testing.assert_allclose(R.gaussian_filter(x, 1.2, 5), g[f"gauss_wide{i}"],
                                           rtol=1e-14, atol=1e-12)
            if f"blur_apply{i}" in g:
                op = R.CirculantBlur(R.psf_taps("uniform", 9), shp)
                np.testing.assert_allclose(op.apply(x), g[f"blur_apply{i}"], atol=1e-11)
                np.testing.assert_allclose(op.adjoint(x), g[f"blur_adjoint{i}"], atol=1e-11)
            if f"bd_apply{i}" in g:
                op = R.BlurDecimate(R.psf_taps("gaussian", 7, 1.6), 3, shp)
                np.testing.assert_allclose(op.apply(x), g[f"bd_apply{i}"], atol=1e-11)
                np.testing.assert_allclose(op.adjoint(g[f"bd_z{i}"]), g[f"bd_adjoint{i}"], atol=1e-12)
            if f"patch{i}" in g:
                np.testing.assert_allclose(R.patch_weighted(x), g[f"patch{i}"], rtol=1e-13, atol=1e-10)
            np.testing.assert_array_equal(extras.median3(x), g[f"median{i}"])
            i += 1
        assert i >= 6

    @pytest.mark.parametrize("shape", [(7, 9), (16, 16), (33, 20)])
    def test_median_matches_scipy_wrap(self, shape):
        x = np.random.default_rng(1).uniform(0, 255, shape)
        np.testing.assert_array_equal(extras.median3(x), ndimage.median_filter(x, size=3, mode="wrap"))
        x32 = x.astype(np.float32)
        np.testing.assert_array_equal(extras.median3(x32).astype(np.float32),
                                      ndimage.median_filter(x32, size=3, mode="wrap"))

    def test_filter_bank_properties(self):
        fb = extras.FilterBank(seed=0)
        x = np.random.default_rng(2).uniform(0, 255, (20, 24))
        assert np.allclose(fb(np.full((8, 8), 77.0)), 77.0)  # zero-mean filters keep constants
        assert np.abs(fb.k.sum(axis=(1, 2))).max() < 1e-12
        # adjointness of the corr/conv pair used by the stage
        k = fb.k[0]
        z = np.random.default_rng(3).standard_normal(x.shape)
        lhs = np.vdot(extras._corr_periodic(x, k), z)
        rhs = np.vdot(x, extras._conv_periodic(z, k))
        assert abs(lhs - rhs) <= 1e-9 * abs(lhs)


class TestDeblurTraces:
    @pytest.mark.parametrize("name,method,m,kappa,budget,stab", [
        ("fp", None, 0, 5, 60, 0), ("mpe", "mpe", 0, 5, 60, 0), ("rre", "rre", 0, 5, 60, 0),
        ("svdmpe", "svdmpe", 0, 5, 60, 0), ("mpe_m2k3", "mpe", 2, 3, 40, 3)])
    def test_g32(self, golden, name, method, m, kappa, budget, stab):
        g = golden("deblur_traces.npz")
        truth, y = g["g32/truth"], g["g32/y"]
        op = R.CirculantBlur(R.psf_taps("uniform", 9), truth.shape)
        red = R.Red(op, y, SQRT2, 0.02, R.gaussian_filter)
        step, cost = R.red_problem(red)
        if method is None:
            x, tr = R.run_fp(step, y, budget, objective=cost, reference=truth.ravel())
        else:
            x, tr = R.run_cycling(step, y, budget, method, m, kappa, objective=cost,
                                  reference=truth.ravel(), stabilization=stab)
        assert _rel(x, g[f"g32/{name}/x"]) <= 1e-11
        _trace_close(tr, g, f"g32/{name}")

    @pytest.mark.parametrize("name,method", [("fp", None), ("mpe", "mpe"), ("rre", "rre")])
    def test_median64(self, golden, name, method):
        g = golden("deblur_traces.npz")
        truth, y = g["m64/truth"], g["m64/y"]
        op = R.CirculantBlur(R.psf_taps("uniform", 9), truth.shape)
        red = R.Red(op, y, SQRT2, 0.02, extras.median3)
        step, cost = R.red_problem(red)
        if method is None:
            x, tr = R.run_fp(step, y, 40, objective=cost, reference=truth.ravel())
        else:
            x, tr = R.run_cycling(step, y, 40, method, objective=cost, reference=truth.ravel())
        assert _rel(x, g[f"m64/{name}/x"]) <= 1e-11
        _trace_close(tr, g, f"m64/{name}")


class TestSuperres:
    def test_step_and_ragged(self, golden):
        g = golden("superres.npz")
        truth, y, x0 = g["sr48/truth"], g["sr48/y"], g["sr48/x0"]
        op = R.BlurDecimate(R.psf_taps("gaussian", 7, 1.6), 3, truth.shape)
        np.testing.assert_allclose(op.adjoint(y), x0, atol=1e-12)
        red = R.Red(op, y, 5.0, 0.02, R.patch_weighted)
        assert _rel(red.fp_step(x0), g["sr48/step1"]) <= 1e-12
        t2 = g["sr_ragged/truth"]
        op2 = R.BlurDecimate(R.psf_taps("gaussian", 7, 1.6), 3, t2.shape)
        red2 = R.Red(op2, g["sr_ragged/y"], 5.0, 0.02, R.gaussian_filter)
        assert _rel(red2.fp_step(g["sr_ragged/x"]), g["sr_ragged/step"]) <= 1e-12

    @pytest.mark.parametrize("name,method", [("fp", None), ("rre", "rre")])
    def test_sr48_trace(self, golden, name, method):
        g = golden("superres.npz")
        truth, y, x0 = g["sr48/truth"], g["sr48/y"], g["sr48/x0"]
        op = R.BlurDecimate(R.psf_taps("gaussian", 7, 1.6), 3, truth.shape)
        red = R.Red(op, y, 5.0, 0.02, R.patch_weighted)
        step, cost = R.red_problem(red)
        if method is None:
            x, tr = R.run_fp(step, x0, 30, objective=cost, reference=truth.ravel())
        else:
            x, tr = R.run_cycling(step, x0, 30, method, objective=cost, reference=truth.ravel())
        assert _rel(x, g[f"sr48/{name}/x"]) <= 1e-10
        _trace_close(tr, g, f"sr48/{name}", rtol=1e-9)


def test_product_filter_bank_params_match_oracle():
    """The product draws the seeded filter-bank parameters itself; they must be
    bit-identical to the oracle's (host-side, CPU test)."""
    from paper_1805_02158_b200.denoisers import filter_bank_params

    for seed in (0, 1, 7):
        k, s, tau = filter_bank_params(seed)
        ko, so, tauo = extras.filter_bank_params(seed)
        np.testing.assert_array_equal(k, ko)
        np.testing.assert_array_equal(s, so)
        assert tau == tauo
