"""Gradient baselines and the remaining reference tasks on the device.

* SD / SD-VE / Nesterov (solvers.py:274-337) through ``solve`` on the device
  schedule, against traces from the UNMODIFIED reference
  (tests/golden/make_config_golden.py) and the reference's committed demo
  traces (pkg/demos/out/deblur_{sd,nesterov}.csv -- known-answer tests).
* ``RedObjective.gradient`` (objective.py:90-93) on both operator routes.
* The deblur-gaussian task (cli.py:115-116): fp_step, cost terms, solves.
* Denoiser condition checkers (objective.py:153-184) over device denoisers.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SQRT2 = float(np.sqrt(2.0))


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def rv():
    import paper_1805_02158_b200 as rv

    return rv


from trace_cmp import cmp_trace  # noqa: E402


def g32_problem(rv, g):
    truth, y = g["g32/truth"], g["g32/y"]
    obj = rv.RedObjective(rv.Blur(rv.make_psf("uniform", 9), truth.shape), y, SQRT2, 0.02,
                          rv.GaussianFilter())
    return obj, rv.as_fixed_point_problem(obj, reference=truth), y


@pytest.mark.parametrize("name,cfg", [
    ("sd", dict(method="sd", max_inner_steps=60)),
    ("nesterov", dict(method="nesterov", max_inner_steps=60)),
    ("sdmpe", dict(method="sd-ve", ve_method="mpe", m=0, kappa=8, max_inner_steps=60)),
    ("sdrre_stab", dict(method="sd-ve", ve_method="rre", m=1, kappa=4, max_inner_steps=40,
                        stabilization_iters=2)),
])
def test_g32_gradient_methods_vs_reference(rv, golden, name, cfg):
    g = golden("gradient_tasks.npz")
    obj, prob, y = g32_problem(rv, g)
    conf = rv.SolveConfig(step_size=rv.default_step_size(SQRT2, 0.02), **cfg)
    assert prob.red.device_solvable
    x, tr = rv.solve(prob, y.ravel(), conf)
    assert rel(x, g[f"g32/{name}/x"]) <= 1e-5
    # SD-MPE with kappa = 8: the windows' pivot ratios reach ~2e-7 (cond(R) ~ 1e7),
    # and the reference itself moves its costs by 1.9e-5 (x by 8e-6) when its
    # windows are perturbed by 1e-15 relative (/tmp experiment recorded in
    # DESIGN.md section 4): costs are compared at the reference's own resolution
    if name == "sdmpe":  # the reference's own resolution (see above)
        cmp_trace(tr, g, f"g32/{name}", cost_rtol=1e-4, sn_rtol=1e-4, sn_atol=1e-5,
                  sig_floor=1e-5)
    else:
        cmp_trace(tr, g, f"g32/{name}")


@pytest.mark.parametrize("name,run", [("sd", "run_steepest_descent"), ("nesterov", "run_nesterov")])
def test_demo64_known_answer(rv, golden, name, run):
    """pkg/demos/02_deblurring.py's committed SD / Nesterov traces (64^2, budget 120)."""
    g = golden("demo64.npz")
    truth, y = g["truth"], g["y"]
    obj = rv.RedObjective(rv.Blur(rv.make_psf("uniform", 9), truth.shape), y, SQRT2, 0.02,
                          rv.GaussianFilter())
    prob = rv.as_fixed_point_problem(obj, reference=truth)
    cfg = rv.SolveConfig(method=name, step_size=rv.default_step_size(SQRT2, 0.02),
                         max_inner_steps=120)
    _, tr = getattr(rv, run)(prob, y.ravel(), cfg)
    np.testing.assert_array_equal([r.iter for r in tr.records], g[f"{name}/iter"])
    np.testing.assert_allclose(tr.costs(), g[f"{name}/cost"], rtol=1e-10)
    np.testing.assert_allclose(tr.step_norms(), g[f"{name}/step_norm"], rtol=1e-7)
    ps = np.array([r.psnr for r in tr.records])
    np.testing.assert_allclose(ps, g[f"{name}/psnr"], atol=1e-9)


def test_gradient_values(rv, golden):
    g = golden("gradient_tasks.npz")
    obj, _, y = g32_problem(rv, g)
    assert rel(obj.gradient(y), g["g32/grad_y"]) <= 1e-12
    t48, y48, x48 = g["sr48/truth"], g["sr48/y"], g["sr48/x0"]
    o48 = rv.RedObjective(rv.BlurDownsample(rv.make_psf("gaussian", 7, 1.6), 3, t48.shape), y48,
                          5.0, 0.02, rv.GaussianFilter())
    assert rel(o48.gradient(x48), g["sr48/grad_x0"]) <= 1e-12


def test_sr48_sd_vs_reference(rv, golden):
    g = golden("gradient_tasks.npz")
    t48, y48, x48 = g["sr48/truth"], g["sr48/y"], g["sr48/x0"]
    obj = rv.RedObjective(rv.BlurDownsample(rv.make_psf("gaussian", 7, 1.6), 3, t48.shape), y48,
                          5.0, 0.02, rv.GaussianFilter())
    prob = rv.as_fixed_point_problem(obj, reference=t48)
    x, tr = rv.solve(prob, x48.ravel(), rv.SolveConfig(
        method="sd", step_size=rv.default_step_size(5.0, 0.02), max_inner_steps=30))
    assert rel(x, g["sr48/sd/x"]) <= 1e-5
    cmp_trace(tr, g, "sr48/sd")


def test_gradient_batch_matches_singles(rv, R):
    """Nesterov on a 3-image batch equals three single solves (per-image masks,
    shared momentum schedule)."""
    from paper_1805_02158_b200.synth import voronoi_scene

    n = 48
    truths = np.stack([voronoi_scene(s, n) for s in range(3)])
    op_o = R.CirculantBlur(R.psf_taps("uniform", 9), (n, n))
    ys = np.stack([R.measure(truths[b], op_o, SQRT2, b) for b in range(3)])
    op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
    cfg = rv.SolveConfig(method="nesterov", step_size=rv.default_step_size(SQRT2, 0.02),
                         max_inner_steps=25)
    X, traces = rv.solve_batch(rv.RedBatch(op, ys, SQRT2, 0.02, rv.Median3()), ys, cfg)
    X = X.cpu().numpy()
    for b in range(3):
        Xb, tb = rv.solve_batch(rv.RedBatch(op, ys[b:b + 1], SQRT2, 0.02, rv.Median3()),
                                ys[b:b + 1], cfg)
        np.testing.assert_array_equal(X[b], Xb.cpu().numpy()[0])
        np.testing.assert_array_equal(traces[b].step_norms(), tb[0].step_norms())


@pytest.fixture(scope="module")
def R():
    from oracle import redve_ref

    return redve_ref


# ----------------------------------------------------------------- deblur-gaussian
def test_deblur_gaussian_task(rv, golden):
    g = golden("gradient_tasks.npz")
    truth, y = g["dg64/truth"], g["dg64/y"]
    obj = rv.RedObjective(rv.Blur(rv.make_psf("gaussian", 9, 1.6), truth.shape), y, SQRT2, 0.02,
                          rv.GaussianFilter())
    assert rel(obj.fp_step(y), g["dg64/step1"]) <= 1e-12
    assert rel(obj.gradient(y), g["dg64/grad_y"]) <= 1e-12
    c = g["dg64/cost_y"]
    np.testing.assert_allclose([obj.cost(y), obj.data_fidelity(y), obj.regularizer(y)], c,
                               rtol=1e-11)
    prob = rv.as_fixed_point_problem(obj, reference=truth)
    for name, cfg in {
        "fp": rv.SolveConfig(method="fp", max_inner_steps=80),
        "mpe": rv.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=80),
        "nesterov": rv.SolveConfig(method="nesterov", step_size=rv.default_step_size(SQRT2, 0.02),
                                   max_inner_steps=80),
    }.items():
        x, tr = rv.solve(prob, y.ravel(), cfg)
        assert rel(x, g[f"dg64/{name}/x"]) <= 1e-5, name
        cmp_trace(tr, g, f"dg64/{name}")


# ----------------------------------------------------------------- condition checkers
@pytest.mark.parametrize("name", ["gauss", "patch", "median"])
def test_condition_checkers_vs_reference(rv, golden, name):
    g = golden("checkers.npz")
    x = g["x"]
    den = {"gauss": rv.GaussianFilter(), "patch": rv.PatchWeighted(), "median": rv.Median3()}[name]
    for c in (0.9, 1.1):
        got = rv.check_local_homogeneity(den, x, c)
        np.testing.assert_allclose(got, g[f"{name}/homog_{c}"], rtol=1e-8, atol=1e-14)
    np.testing.assert_allclose(rv.check_passivity(den, x, iterations=20, seed=0),
                               g[f"{name}/passivity"], rtol=1e-6)
    np.testing.assert_allclose(rv.check_passivity(den, x, iterations=5, seed=3),
                               g[f"{name}/passivity5_s3"], rtol=1e-6)
