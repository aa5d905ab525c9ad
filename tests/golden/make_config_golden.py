"""Config-scale golden fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_config_golden.py [c1] [c2] [c3] [grad] [checkers]

Reads ``/root/reference/pkg/src`` read-only and writes ``tests/golden/config_*.npz``.
Each case runs the reference's own ``RedObjective`` + ``solve`` at a
BASELINE.json config's full image size.  Inputs are NOT stored: the tests
rebuild them with ``synth.voronoi_scene`` + ``oracle.redve_ref.measure``
(bit-identical to ``redve.degrade``, checked here and pinned by the stored
SHA-256 of every measurement).  Solutions are stored as float32 (rounding
6e-8 relative, far below the 1e-5 parity bar); traces as float64.

* c1: configs[1] -- 256^2, 9x9 uniform blur, sigma sqrt(2), 3x3 median plugged
  into the reference through its callable-denoiser protocol, FP / FP+MPE /
  FP+RRE, 200 iterations; four images spread over the 64-image bench batch.
* c2: configs[2] -- 768^2 SR x3 (7x7 Gaussian 1.6), sigma 5, PatchWeighted,
  x0 = H^T y, FP+RRE with budget 7 (one full cycle + one step) and FP with
  budget 5; scipy ``cg`` wrapped to count its iterations per fixed-point step.
* c3: configs[3] -- 512^2, FilterBank (oracle/extras, parity of the denoiser
  itself unpinned) inside the reference drivers, FP+MPE 24 iterations, 2 images.
* grad: SD / SD-VE / Nesterov on 32^2 (GaussianFilter) and the deblur-gaussian
  task (cli.py:115-116) FP / FP+MPE on 64^2, plus its fp_step and gradient.
* checkers: check_local_homogeneity / check_passivity (objective.py:153-184).
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import redve  # noqa: E402  (the reference)
import redve.objective as robj  # noqa: E402
from redve.objective import as_fixed_point_problem, default_step_size  # noqa: E402

from oracle import extras  # noqa: E402
from oracle import redve_ref as R  # noqa: E402
from paper_1805_02158_b200.synth import voronoi_scene  # noqa: E402

SQRT2 = float(np.sqrt(2.0))
C1_SEEDS = (0, 21, 42, 63)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def trace_arrays(trace):
    nan = lambda v: np.nan if v is None else v
    cw = trace.cycle_weights
    return dict(
        iter=np.array([r.iter for r in trace.records], dtype=np.int64),
        cost=np.array([nan(r.cost) for r in trace.records]),
        psnr=np.array([nan(r.psnr) for r in trace.records]),
        step_norm=np.array([r.step_norm for r in trace.records]),
        gamma_abs_sum=np.array([nan(r.gamma_abs_sum) for r in trace.records]),
        n_cycles=np.int64(len(cw)),
        cycle_stability=np.array([w.stability_sum for w in cw]),
        cycle_fallback=np.array([0 if w.fallback_from is None else 1 for w in cw], dtype=np.int64),
    )


def _store(out, key, sol, trace):
    out[f"{key}/x32"] = np.asarray(sol, dtype=np.float32)
    out[f"{key}/xnorm"] = np.float64(np.linalg.norm(sol))
    for k, v in trace_arrays(trace).items():
        out[f"{key}/{k}"] = v


def _deblur_inputs(seed, n, psf=("uniform", 9)):
    truth = voronoi_scene(seed, n)
    op = redve.Blur(redve.make_psf(*psf), truth.shape)
    y = redve.degrade(truth, op, SQRT2, seed=seed)
    taps = R.psf_taps(*psf) if len(psf) == 2 else R.psf_taps(psf[0], psf[1], psf[2])
    y_or = R.measure(truth, R.CirculantBlur(taps, truth.shape), SQRT2, seed)
    assert np.array_equal(y, y_or), "oracle measurement differs from redve.degrade"
    return truth, op, y


def config1():
    out = {"seeds": np.array(C1_SEEDS)}
    for seed in C1_SEEDS:
        truth, op, y = _deblur_inputs(seed, 256)
        out[f"s{seed}/y_sha"] = np.array(sha(y))
        obj = redve.RedObjective(forward=op, y=y, sigma=SQRT2, alpha=0.02, denoiser=extras.median3)
        prob = as_fixed_point_problem(obj, reference=truth)
        for name, cfg in {
            "fp": redve.SolveConfig(method="fp", max_inner_steps=200),
            "mpe": redve.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=200),
            "rre": redve.SolveConfig(method="fp-ve", ve_method="rre", max_inner_steps=200),
        }.items():
            sol, tr = redve.solve(prob, y.ravel(), cfg)
            _store(out, f"s{seed}/{name}", sol, tr)
            print("c1", seed, name, tr.records[-1].cost, flush=True)
    np.savez_compressed(os.path.join(HERE, "config_c1.npz"), **out)


class _CountingCg:
    """scipy cg wrapper that logs the iteration count of every call."""

    def __init__(self, cg):
        self.cg, self.counts = cg, []

    def __call__(self, *args, **kw):
        n = [0]
        user_cb = kw.pop("callback", None)

        def cb(xk):
            n[0] += 1
            if user_cb is not None:
                user_cb(xk)

        res = self.cg(*args, callback=cb, **kw)
        self.counts.append(n[0])
        return res


def config2():
    out = {}
    truth = voronoi_scene(0, 768)
    op = redve.BlurDownsample(redve.make_psf("gaussian", 7, 1.6), 3, truth.shape)
    y = redve.degrade(truth, op, 5.0, seed=0)
    y_or = R.measure(truth, R.BlurDecimate(R.psf_taps("gaussian", 7, 1.6), 3, truth.shape), 5.0, 0)
    assert np.array_equal(y, y_or)
    out["y_sha"] = np.array(sha(y))
    x0 = op.adjoint(y)
    orig = robj.cg
    try:
        for name, cfg in {
            "fp5": redve.SolveConfig(method="fp", max_inner_steps=5),
            "rre7": redve.SolveConfig(method="fp-ve", ve_method="rre", max_inner_steps=7),
        }.items():
            counter = _CountingCg(orig)
            robj.cg = counter
            obj = redve.RedObjective(forward=op, y=y, sigma=5.0, alpha=0.02,
                                     denoiser=redve.PatchWeighted())
            prob = as_fixed_point_problem(obj, reference=truth)
            sol, tr = redve.solve(prob, x0.ravel(), cfg)
            _store(out, name, sol, tr)
            out[f"{name}/cg_iters"] = np.array(counter.counts, dtype=np.int64)
            print("c2", name, counter.counts, tr.records[-1].cost, flush=True)
    finally:
        robj.cg = orig
    np.savez_compressed(os.path.join(HERE, "config_c2.npz"), **out)


def config3():
    out = {}
    bank = extras.FilterBank(0)
    for seed in (0, 1):
        truth, op, y = _deblur_inputs(seed, 512)
        out[f"s{seed}/y_sha"] = np.array(sha(y))
        obj = redve.RedObjective(forward=op, y=y, sigma=SQRT2, alpha=0.02, denoiser=bank)
        prob = as_fixed_point_problem(obj, reference=truth)
        sol, tr = redve.solve(prob, y.ravel(),
                              redve.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=24))
        _store(out, f"s{seed}/mpe", sol, tr)
        print("c3", seed, tr.records[-1].cost, flush=True)
    np.savez_compressed(os.path.join(HERE, "config_c3.npz"), **out)


def gradient_and_tasks():
    out = {}
    truth = redve.synthetic_image(32)
    op = redve.Blur(redve.make_psf("uniform", 9), truth.shape)
    y = redve.degrade(truth, op, SQRT2, seed=0)
    out["g32/truth"], out["g32/y"] = truth, y
    obj = redve.RedObjective(forward=op, y=y, sigma=SQRT2, alpha=0.02, denoiser=redve.GaussianFilter())
    prob = as_fixed_point_problem(obj, reference=truth)
    step = default_step_size(SQRT2, 0.02)
    out["g32/grad_y"] = obj.gradient(y)
    for name, cfg in {
        "sd": redve.SolveConfig(method="sd", step_size=step, max_inner_steps=60),
        "nesterov": redve.SolveConfig(method="nesterov", step_size=step, max_inner_steps=60),
        "sdmpe": redve.SolveConfig(method="sd-ve", ve_method="mpe", m=0, kappa=8, step_size=step,
                                   max_inner_steps=60),
        "sdrre_stab": redve.SolveConfig(method="sd-ve", ve_method="rre", m=1, kappa=4,
                                        step_size=step, max_inner_steps=40, stabilization_iters=2),
    }.items():
        sol, tr = redve.solve(prob, y.ravel(), cfg)
        out[f"g32/{name}/x"] = sol
        for k, v in trace_arrays(tr).items():
            out[f"g32/{name}/{k}"] = v
    # superres gradient (CG-route operator) on 48^2 with the Gaussian denoiser
    t48 = redve.synthetic_image(48)
    bd = redve.BlurDownsample(redve.make_psf("gaussian", 7, 1.6), 3, t48.shape)
    y48 = redve.degrade(t48, bd, 5.0, seed=0)
    o48 = redve.RedObjective(forward=bd, y=y48, sigma=5.0, alpha=0.02, denoiser=redve.GaussianFilter())
    x48 = bd.adjoint(y48)
    out["sr48/truth"], out["sr48/y"], out["sr48/x0"] = t48, y48, x48
    out["sr48/grad_x0"] = o48.gradient(x48)
    p48 = as_fixed_point_problem(o48, reference=t48)
    sol, tr = redve.solve(p48, x48.ravel(), redve.SolveConfig(
        method="sd", step_size=default_step_size(5.0, 0.02), max_inner_steps=30))
    out["sr48/sd/x"] = sol
    for k, v in trace_arrays(tr).items():
        out[f"sr48/sd/{k}"] = v
    # deblur-gaussian task (cli.py:115-116): 9x9 Gaussian PSF std 1.6
    truth = redve.synthetic_image(64)
    op = redve.Blur(redve.make_psf("gaussian", 9, 1.6), truth.shape)
    y = redve.degrade(truth, op, SQRT2, seed=1)
    out["dg64/truth"], out["dg64/y"] = truth, y
    obj = redve.RedObjective(forward=op, y=y, sigma=SQRT2, alpha=0.02, denoiser=redve.GaussianFilter())
    out["dg64/step1"] = obj.fp_step(y)
    out["dg64/grad_y"] = obj.gradient(y)
    out["dg64/cost_y"] = np.array([obj.cost(y), obj.data_fidelity(y), obj.regularizer(y)])
    prob = as_fixed_point_problem(obj, reference=truth)
    for name, cfg in {
        "fp": redve.SolveConfig(method="fp", max_inner_steps=80),
        "mpe": redve.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=80),
        "nesterov": redve.SolveConfig(method="nesterov", step_size=default_step_size(SQRT2, 0.02),
                                      max_inner_steps=80),
    }.items():
        sol, tr = redve.solve(prob, y.ravel(), cfg)
        out[f"dg64/{name}/x"] = sol
        for k, v in trace_arrays(tr).items():
            out[f"dg64/{name}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "gradient_tasks.npz"), **out)


def checkers():
    out = {}
    x = redve.synthetic_image(40)
    out["x"] = x
    for name, den in {"gauss": redve.GaussianFilter(), "patch": redve.PatchWeighted(),
                      "median": extras.median3}.items():
        for c in (0.9, 1.1):
            out[f"{name}/homog_{c}"] = np.float64(robj.check_local_homogeneity(den, x, c))
        out[f"{name}/passivity"] = np.float64(robj.check_passivity(den, x, iterations=20, seed=0))
        out[f"{name}/passivity5_s3"] = np.float64(robj.check_passivity(den, x, iterations=5, seed=3))
    np.savez_compressed(os.path.join(HERE, "checkers.npz"), **out)


if __name__ == "__main__":
    want = set(sys.argv[1:]) or {"c1", "c2", "c3", "grad", "checkers"}
    if "grad" in want:
        gradient_and_tasks()
    if "checkers" in want:
        checkers()
    if "c3" in want:
        config3()
    if "c1" in want:
        config1()
    if "c2" in want:
        config2()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
