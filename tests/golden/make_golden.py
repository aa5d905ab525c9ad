"""Generate the golden fixtures by importing the UNMODIFIED reference package.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

Reads ``/root/reference/pkg/src`` read-only and writes ``tests/golden/*.npz``.
Every fixture stores its inputs next to the reference's outputs, so the tests
can replay them with nothing but numpy.  The median / filter-bank cases plug
the in-repo oracles (``oracle/extras.py``) into the reference's own
``RedObjective`` and drivers through its callable-denoiser protocol.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import redve  # noqa: E402  (the reference)
from redve import extrapolation as rve  # noqa: E402
from redve.objective import as_fixed_point_problem  # noqa: E402

from oracle import extras  # noqa: E402
from paper_1805_02158_b200.synth import voronoi_scene  # noqa: E402

SQRT2 = float(np.sqrt(2.0))


def _trace_arrays(trace):
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


def ve_windows():
    """extrapolate_once on hand-built windows covering every branch of
    extrapolation.py:319-386."""
    rng = np.random.default_rng(11)
    cases = {}
    # random full-rank windows, several orders and lengths
    for i, (n, k) in enumerate([(50, 1), (50, 3), (64, 5), (300, 5), (4096, 5), (1000, 8)]):
        cases[f"random{i}"] = rng.standard_normal((k + 2, n))
    # linear fixed-point windows (exactness at the minimal polynomial degree)
    basis, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    a = basis @ np.diag([0.9, 0.9, 0.5, 0.5, 0.1, 0.1]) @ basis.T
    b = rng.standard_normal(6)
    x = np.zeros(6)
    seq = [x]
    for _ in range(8):
        x = a @ x + b
        seq.append(x)
    cases["linear_k3"] = np.array(seq[:5])
    cases["linear_k5_rankdef"] = np.array(seq[:7])
    # rank-1 geometric window at kappa=3 (shrinks to kappa_used=1)
    v = np.array([1.0, 2.0, -1.0, 0.5])
    lim = np.array([10.0, -3.0, 5.0, 2.0])
    cases["rank1"] = np.array([lim + v * 0.6**j for j in range(5)])
    # stationary window
    cases["stationary"] = np.tile(np.array([1.0, -2.0, 3.0]), (4, 1))
    # MPE degenerate sum -> RRE fallback: c = (-1, 1) has sum 0 (u1 = u0 exactly)
    cases["mpe_degenerate"] = np.array([[0.0, 0.0], [1.0, 2.0], [2.0, 4.0 + 1e-3]])
    # near-degenerate oscillation
    cases["oscillating"] = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 0.0]])
    # decaying smooth image-like windows
    xs = [np.cumsum(rng.standard_normal(2048)) for _ in range(1)][0]
    d = rng.standard_normal((6, 2048))
    rates = np.array([0.95, 0.8, 0.6, 0.4, 0.2, 0.1])
    cases["decay_k5"] = np.array([xs + (rates**j) @ d for j in range(7)])
    out = {}
    for name, rows in cases.items():
        out[f"{name}/rows"] = rows
        for method in rve.METHODS:
            res = rve.extrapolate_once(rve.VectorSequenceWindow(rows), method)
            key = f"{name}/{method}"
            out[f"{key}/vector"] = res.vector
            out[f"{key}/flags"] = np.array(
                [int(res.converged), int(res.extrapolated), res.kappa_used,
                 -1 if res.weights is None else int(res.weights.fallback_from is not None)])
            if res.weights is not None:
                out[f"{key}/gamma"] = res.weights.gamma
                out[f"{key}/c"] = res.weights.c
                out[f"{key}/stability"] = np.float64(res.weights.stability_sum)
    np.savez_compressed(os.path.join(HERE, "ve_windows.npz"), **out)


def operators_and_denoisers():
    rng = np.random.default_rng(5)
    out = {}
    shapes = [(8, 8), (12, 10), (16, 16), (24, 24), (33, 20), (64, 64)]
    for i, shp in enumerate(shapes):
        x = rng.uniform(0, 255, shp)
        out[f"x{i}"] = x
        out[f"gauss{i}"] = redve.GaussianFilter()(x)
        out[f"gauss_wide{i}"] = redve.GaussianFilter(1.2, 5)(x) if min(shp) >= 5 else x
        if min(shp) >= 9:
            blur = redve.Blur(redve.make_psf("uniform", 9), shp)
            out[f"blur_apply{i}"] = blur.apply(x)
            out[f"blur_adjoint{i}"] = blur.adjoint(x)
        if min(shp) >= 7:
            bd = redve.BlurDownsample(redve.make_psf("gaussian", 7, 1.6), 3, shp)
            out[f"bd_apply{i}"] = bd.apply(x)
            z = rng.standard_normal(bd.out_shape)
            out[f"bd_z{i}"] = z
            out[f"bd_adjoint{i}"] = bd.adjoint(z)
        if shp[0] * shp[1] <= 1024:
            out[f"patch{i}"] = redve.PatchWeighted()(x)
        out[f"median{i}"] = extras.median3(x)
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **out)


def deblur_traces():
    """Deblur FP / FP+VE traces through the reference drivers."""
    out = {}
    # 32^2, GaussianFilter: cost logged every step (N <= 128^2)
    truth = redve.synthetic_image(32)
    op = redve.Blur(redve.make_psf("uniform", 9), truth.shape)
    y = redve.degrade(truth, op, SQRT2, seed=0)
    out["g32/truth"], out["g32/y"] = truth, y
    obj = redve.RedObjective(forward=op, y=y, sigma=SQRT2, alpha=0.02, denoiser=redve.GaussianFilter())
    prob = as_fixed_point_problem(obj, reference=truth)
    runs = {
        "fp": redve.SolveConfig(method="fp", max_inner_steps=60),
        "mpe": redve.SolveConfig(method="fp-ve", ve_method="mpe", m=0, kappa=5, max_inner_steps=60),
        "rre": redve.SolveConfig(method="fp-ve", ve_method="rre", m=0, kappa=5, max_inner_steps=60),
        "svdmpe": redve.SolveConfig(method="fp-ve", ve_method="svdmpe", m=0, kappa=5, max_inner_steps=60),
        "mpe_m2k3": redve.SolveConfig(method="fp-ve", ve_method="mpe", m=2, kappa=3, max_inner_steps=40,
                                      stabilization_iters=3),
    }
    for name, cfg in runs.items():
        sol, tr = redve.solve(prob, y.ravel(), cfg)
        out[f"g32/{name}/x"] = sol
        for k, v in _trace_arrays(tr).items():
            out[f"g32/{name}/{k}"] = v

    # 64^2 Voronoi scene, median denoiser plugged into the reference
    truth = voronoi_scene(3, 64)
    op = redve.Blur(redve.make_psf("uniform", 9), truth.shape)
    y = redve.degrade(truth, op, SQRT2, seed=3)
    out["m64/truth"], out["m64/y"] = truth, y
    obj = redve.RedObjective(forward=op, y=y, sigma=SQRT2, alpha=0.02, denoiser=extras.median3)
    prob = as_fixed_point_problem(obj, reference=truth)
    for name, cfg in {
        "fp": redve.SolveConfig(method="fp", max_inner_steps=40),
        "mpe": redve.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=40),
        "rre": redve.SolveConfig(method="fp-ve", ve_method="rre", max_inner_steps=40),
    }.items():
        sol, tr = redve.solve(prob, y.ravel(), cfg)
        out[f"m64/{name}/x"] = sol
        for k, v in _trace_arrays(tr).items():
            out[f"m64/{name}/{k}"] = v

    # config-0 shape: 256^2 Voronoi, GaussianFilter, FP+MPE, budget 200 (cost every 5th)
    truth = voronoi_scene(0, 256)
    op = redve.Blur(redve.make_psf("uniform", 9), truth.shape)
    y = redve.degrade(truth, op, SQRT2, seed=0)
    out["c0/truth"], out["c0/y"] = truth, y
    obj = redve.RedObjective(forward=op, y=y, sigma=SQRT2, alpha=0.02, denoiser=redve.GaussianFilter())
    prob = as_fixed_point_problem(obj, reference=truth)
    for name, cfg in {
        "fp": redve.SolveConfig(method="fp", max_inner_steps=200),
        "mpe": redve.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=200),
    }.items():
        sol, tr = redve.solve(prob, y.ravel(), cfg)
        out[f"c0/{name}/x"] = sol
        for k, v in _trace_arrays(tr).items():
            out[f"c0/{name}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "deblur_traces.npz"), **out)


def superres_traces():
    """SR x3 (CG data term, PatchWeighted) at 48^2 -- AC8 analog, smaller."""
    out = {}
    truth = redve.synthetic_image(48)
    op = redve.BlurDownsample(redve.make_psf("gaussian", 7, 1.6), 3, truth.shape)
    y = redve.degrade(truth, op, 5.0, seed=0)
    x0 = op.adjoint(y)
    out["sr48/truth"], out["sr48/y"], out["sr48/x0"] = truth, y, x0
    obj = redve.RedObjective(forward=op, y=y, sigma=5.0, alpha=0.02, denoiser=redve.PatchWeighted())
    out["sr48/step1"] = obj.fp_step(x0)
    prob = as_fixed_point_problem(obj, reference=truth)
    for name, cfg in {
        "fp": redve.SolveConfig(method="fp", max_inner_steps=30),
        "rre": redve.SolveConfig(method="fp-ve", ve_method="rre", max_inner_steps=30),
    }.items():
        sol, tr = redve.solve(prob, x0.ravel(), cfg)
        out[f"sr48/{name}/x"] = sol
        for k, v in _trace_arrays(tr).items():
            out[f"sr48/{name}/{k}"] = v
    # CG with the Gaussian denoiser on a ragged shape (ceil out_shape)
    truth = redve.synthetic_image(20, 26)
    op = redve.BlurDownsample(redve.make_psf("gaussian", 7, 1.6), 3, truth.shape)
    y = redve.degrade(truth, op, 5.0, seed=4)
    obj = redve.RedObjective(forward=op, y=y, sigma=5.0, alpha=0.02, denoiser=redve.GaussianFilter())
    out["sr_ragged/truth"], out["sr_ragged/y"] = truth, y
    out["sr_ragged/x"] = truth * 0.9
    out["sr_ragged/step"] = obj.fp_step(truth * 0.9)
    np.savez_compressed(os.path.join(HERE, "superres.npz"), **out)


def demo_csv():
    """The reference's committed demo traces (pkg/demos/out/deblur_{fp,fp-mpe}.csv,
    64^2 synthetic_image, 9x9 uniform, sigma=sqrt(2), seed 0, GaussianFilter,
    alpha=0.02, budget 120; pkg/demos/02_deblurring.py:38-61) as arrays."""
    out = {}
    truth = redve.synthetic_image(64)
    op = redve.Blur(redve.make_psf("uniform", 9), truth.shape)
    out["truth"] = truth
    out["y"] = redve.degrade(truth, op, SQRT2, seed=0)
    for name in ("fp", "fp-mpe", "sd", "nesterov"):
        path = f"/root/reference/pkg/demos/out/deblur_{name}.csv"
        raw = open(path, "rb").read()
        out[f"{name}/csv_bytes"] = np.frombuffer(raw, dtype=np.uint8)
        rows = raw.decode("ascii").strip().splitlines()[1:]
        cols = list(zip(*[r.split(",") for r in rows]))
        num = lambda c: np.array([np.nan if v == "" else float(v) for v in c])
        out[f"{name}/iter"] = np.array([int(v) for v in cols[0]])
        out[f"{name}/cost"] = num(cols[1])
        out[f"{name}/psnr"] = num(cols[2])
        out[f"{name}/step_norm"] = num(cols[3])
        out[f"{name}/gamma_abs_sum"] = num(cols[4])
    np.savez_compressed(os.path.join(HERE, "demo64.npz"), **out)


if __name__ == "__main__":
    sections = {"demo": demo_csv, "ve": ve_windows, "ops": operators_and_denoisers,
                "deblur": deblur_traces, "superres": superres_traces}
    for key in (sys.argv[1:] or list(sections)):
        sections[key]()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
