#!/usr/bin/env python
"""Benchmark: RED-FP+MPE image solves/s, BASELINE.json configs[1] workload.

Workload (one "step"): a batch of 64 seeded 256x256 Voronoi scenes, 9x9
uniform circular blur, noise sigma = sqrt(2), 3x3 median denoiser,
alpha = 0.02, FP+MPE with m = 0, kappa = 5, 200 baseline evaluations, tol 0
(the reference defaults, cli.py:60-61,126-129,148), fp64 throughout.  Each
GPU solves its own batch (weak scaling, no collectives: the images are
independent).  The timed region is the device-resident solve of the batch
(inputs already in HBM); ``e2e`` is the same metric through the public API
with host numpy buffers (problem setup + H2D + solve + D2H of solutions and
traces inside the timed region).

``--impl reference`` times the CPU restatement of the reference
(oracle/redve_ref.py + oracle/extras.median3) on the host cores: one image
per core per step, a process pool over every core.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

SIZE, BATCH, BUDGET, KAPPA, ALPHA = 256, 64, 200, 5, 0.02
SIGMA = float(np.sqrt(2.0))
METRIC = "RED-FP+MPE image solves/sec (256^2 deblur)"
WORKLOAD = ("configs[1]: 64 x 256^2 Voronoi scenes, 9x9 uniform blur, sigma=sqrt(2), "
            "3x3 median denoiser, FP+MPE m=0 kappa=5, 200 iterations, fp64")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--cpu-images", type=int, default=4, help="cpu_baseline sample (images)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def make_inputs_cpu(seeds):
    """Seeded scenes and measurements for the CPU legs (oracle ops)."""
    from oracle import redve_ref as R
    from paper_1805_02158_b200.synth import voronoi_scene

    op = R.CirculantBlur(R.psf_taps("uniform", 9), (SIZE, SIZE))
    truths = np.stack([voronoi_scene(int(s), SIZE) for s in seeds])
    ys = np.stack([R.measure(truths[i], op, SIGMA, int(s)) for i, s in enumerate(seeds)])
    return truths, ys


def make_inputs_gpu(seeds):
    """Same scenes and seeded noise through the product API (blur on the GPU)."""
    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200.synth import voronoi_scene

    op = rv.Blur(rv.make_psf("uniform", 9), (SIZE, SIZE))
    truths = np.stack([voronoi_scene(int(s), SIZE) for s in seeds])
    clean = op.apply(truths)
    ys = np.stack([clean[i] + rv.gaussian_noise((SIZE, SIZE), SIGMA, int(s))
                   for i, s in enumerate(seeds)])
    return truths, ys


# ----------------------------------------------------------------------------- CPU side
def _oracle_solve(args):
    seed, y = args
    from oracle import extras
    from oracle import redve_ref as R

    op = R.CirculantBlur(R.psf_taps("uniform", 9), (SIZE, SIZE))
    red = R.Red(op, y, SIGMA, ALPHA, extras.median3)
    step, cost = R.red_problem(red)
    x, tr = R.run_cycling(step, y, BUDGET, "mpe", 0, KAPPA, objective=cost)
    return len(tr.iters)


def _single_thread_env():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"


def cpu_baseline(n_images):
    """Oracle port, 1 core, n_images sequential solves -> solves/s."""
    _, ys = make_inputs_cpu(range(n_images))
    t0 = time.perf_counter()
    for i in range(n_images):
        _oracle_solve((i, ys[i]))
    dt = time.perf_counter() - t0
    return {"value": n_images / dt, "unit": "solves/s", "cores": 1, "kind": "port",
            "sample": f"{n_images} images of the workload solved sequentially (200 iters each) "
                      f"by oracle/redve_ref.py, 1 thread, {dt:.1f} s"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _single_thread_env()
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    _, ys = make_inputs_cpu(range(cores))
    work = [(i, ys[i]) for i in range(cores)]
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores) as pool:
        for it in range(a.warmup + a.steps):
            t0 = time.perf_counter()
            pool.map(_oracle_solve, work, chunksize=1)
            dt = time.perf_counter() - t0
            if it >= a.warmup:
                times.append(dt)
    ms = 1e3 * statistics.mean(times)
    value = cores / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": f"{cores} images per step, one per core"},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "port",
                         "sample": f"{cores} images per step (one per core, process pool), "
                                   "oracle/redve_ref.py restatement of the reference"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU side
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(kind, B, N, s=8, kp1=KAPPA + 1):
    """Bytes each kernel must move per launch (each logical array read/written once)."""
    table = {
        "row_fwd": 2 * B * N * s,            # read x, write the pair spectrum
        "col": 2 * B * N * s + N * 8,        # read+write the spectrum, read g
        "row_inv": 4 * B * N * s,            # read spectrum, x_b, x_prev; write x+
        "cost": 3 * B * N * s,               # read x, y, reference
        "copy_view": 2 * B * N * s,
        "gram": (kp1 + 1) * B * N * s,       # kappa+2 window iterates
        "combine": (kp1 + 1) * B * N * s,    # kappa+1 iterates read, 1 written
        "gather": 2 * B * N * s,
    }
    return table.get(kind)


def measured_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kind):
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    v = d.get(kind)
    return None if v is None else float(v)


def run_native(a):
    import torch
    import torch.distributed as dist

    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200 import _native as nat

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, N = a.batch, SIZE * SIZE
    seeds = range(rank * B, rank * B + B)
    truths, ys = make_inputs_gpu(seeds)
    op = rv.Blur(rv.make_psf("uniform", 9), (SIZE, SIZE))
    cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", m=0, kappa=KAPPA, max_inner_steps=BUDGET)
    y_dev = torch.from_numpy(ys).cuda()
    batch = rv.RedBatch(op, y_dev, SIGMA, ALPHA, rv.Median3())
    x0 = y_dev.clone()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(a.warmup):
        batch.solve(x0, cfg)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    l0 = nat.kernel_launches()
    e0.record(stream)
    for _ in range(a.steps):
        res = batch.solve(x0, cfg)
    e1.record(stream)
    torch.cuda.synchronize()
    l1 = nat.kernel_launches()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / a.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B / (ms / 1e3)
    launches = (l1 - l0) // a.steps
    assert int(res.n_records.min()) == BUDGET and int((res.status != 0).sum()) == 0

    # ---- per-kernel device times (CUDA events bracketing every launch, one extra solve)
    nat.profile(True)
    batch.solve(x0, cfg)
    rep = nat.profile_report()
    nat.profile(False)
    kernels = {}
    for kind, (tot, cnt) in rep.items():
        ab = algorithmic_bytes(kind, B, N)
        avg = tot / cnt
        kernels[kind] = {"launches": cnt, "avg_us": 1e3 * avg, "total_ms": tot,
                         "gbs": None if ab is None else ab / (avg / 1e3) / 1e9}
    step_kernel_ms = sum(v["total_ms"] for v in kernels.values())
    dom = max(kernels, key=lambda k: kernels[k]["total_ms"])
    peak, peak_src = measured_peak()
    ach = kernels[dom]["gbs"]
    roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": None if ach is None else ach / peak, "peak_source": peak_src,
            "share_of_step": kernels[dom]["total_ms"] / step_kernel_ms,
            "algorithmic_bytes_per_launch": algorithmic_bytes(dom, B, N),
            "traffic": ncu_traffic(dom)}

    # ---- e2e through the public API with host buffers (pinned, allocated up front):
    # problem setup from the host measurements, H2D of y and x0, the solve, D2H of
    # the solutions (traces come back inside solve_batch)
    ys_host = torch.from_numpy(ys).pin_memory()
    x_host = torch.empty_like(ys_host).pin_memory()
    e2e_steps = max(1, min(a.steps, 3))
    b2 = rv.RedBatch(op, ys_host, SIGMA, ALPHA, rv.Median3())  # warm the buffer cache
    rv.solve_batch(b2, ys_host, cfg)
    del b2
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        b2 = rv.RedBatch(op, ys_host, SIGMA, ALPHA, rv.Median3())
        X, traces = rv.solve_batch(b2, ys_host, cfg)
        x_host.copy_(X)
        del b2
    Xh = x_host.numpy()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s = float(tt.item())
    assert Xh.shape == (B, SIZE, SIZE) and len(traces) == B
    h2d = 2 * B * N * 8          # measurements for the problem + x0
    d2h = B * N * 8 + B * (BUDGET * 5 * 8)  # solutions + per-record trace arrays

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        _single_thread_env()
        cpu = cpu_baseline(a.cpu_images)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": world * B, "images_per_gpu": B,
                       "image": f"{SIZE}x{SIZE}", "iterations": BUDGET, "parallelism": f"dp{world}",
                       "l2": "working set > L2 (7-slot ring x 64 images = 229 MB)"},
            "e2e": {"value": world * B / e2e_s, "unit": "solves/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s},
            "gpu_launches": int(launches),
            "roofline": roof,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_native(a)


if __name__ == "__main__":
    main()
