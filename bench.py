#!/usr/bin/env python
"""Benchmark: RED-FP+MPE image solves/s on the BASELINE.json configs.

Default workload (one "step", BASELINE.json configs[1], the metric's config):
a batch of 64 seeded 256x256 Voronoi scenes, 9x9 uniform circular blur, noise
sigma = sqrt(2), 3x3 median denoiser, alpha = 0.02, FP+MPE with m = 0,
kappa = 5, 200 baseline evaluations, tol 0 (the reference defaults,
cli.py:60-61,126-129,148), fp64 throughout.  Each GPU solves its own batch
(weak scaling, no collectives: the images are independent).  The timed
region is the device-resident solve of the batch (inputs already in HBM);
``e2e`` is the same metric through the public API from pinned host buffers
(problem setup + H2D + solve + D2H of solutions; traces come back inside).

``--config 0|2|3`` measures the other single-GPU configs with the same
contract (configs[0]: one 256^2 image, GaussianFilter; configs[2]: one 768^2
super-resolution x3 image, PatchWeighted, FP+RRE with the CG data term;
configs[3]: 512 images of 512^2 with the seeded filter-bank denoiser, split
across the ranks).

``--impl reference`` times the reference's CPU path on the host cores: the
UNMODIFIED reference package ``redve`` (pip-installed into baseline/_ref) with
the configs' denoisers plugged in through its callable protocol, the whole
batch per step over a process pool of every core; the oracle restatement
(oracle/redve_ref.py) only when baseline/_ref is absent.

``--gpus N`` outside torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU).
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

BUDGET, KAPPA, ALPHA = 200, 5, 0.02
SQ2 = float(np.sqrt(2.0))
METRIC = "RED-FP+MPE image solves/sec (256^2 deblur)"
SPATIAL_METRIC = "RED-FP+RRE fixed-point iterations/sec (configs[4], 8192^2 SR x3, one image)"

CONFIGS = {
    0: dict(size=256, batch=1, kind="deblur", den="gaussian", sigma=SQ2, ve="mpe", scaling="weak",
            workload="configs[0]: one 256^2 Voronoi scene, 9x9 uniform blur, sigma=sqrt(2), "
                     "GaussianFilter(0.55,5), FP+MPE m=0 kappa=5, 200 iterations, fp64"),
    1: dict(size=256, batch=64, kind="deblur", den="median", sigma=SQ2, ve="mpe", scaling="weak",
            workload="configs[1]: 64 x 256^2 Voronoi scenes, 9x9 uniform blur, sigma=sqrt(2), "
                     "3x3 median denoiser, FP+MPE m=0 kappa=5, 200 iterations, fp64"),
    2: dict(size=768, batch=1, kind="sr", den="patch", sigma=5.0, ve="rre", scaling="weak",
            pw_weights="float32",
            workload="configs[2]: one 768^2 Voronoi scene, 7x7 Gaussian blur std 1.6, x3 decimation, "
                     "sigma=5, PatchWeighted (fp32 weight planes, fp64 arithmetic), FP+RRE m=0 "
                     "kappa=5 with CG, 200 iterations, fp64"),
    3: dict(size=512, batch=512, kind="deblur", den="filterbank", sigma=SQ2, ve="mpe",
            scaling="strong",
            workload="configs[3]: 512 x 512^2 Voronoi scenes split across the GPUs, 9x9 uniform "
                     "blur, sigma=sqrt(2), seeded 8x5x5 filter bank, FP+MPE, 200 iterations, fp64"),
    4: dict(size=8192, batch=1, kind="sr", den="patch", sigma=5.0, ve="rre", scaling="strong",
            pw_weights="float32",
            workload="configs[4]: one 8192^2 Voronoi scene (LR 2731^2), 7x7 Gaussian blur std 1.6, "
                     "x3 decimation, sigma=5, PatchWeighted (fp32 weight planes, fp64 arithmetic), "
                     "FP+RRE m=0 kappa=5 with CG, fp64; "
                     "row slabs across the GPUs with halo exchange + allreduced inner products; "
                     "one step = the first 7 fixed-point iterations + 1 extrapolation"),
}
SPATIAL_BUDGET = 7


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=None, help="override the config's batch")
    ap.add_argument("--cpu-images", type=int, default=4, help="cpu_baseline sample (images)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- inputs
def make_inputs_gpu(c, seeds):
    """Seeded scenes and measurements through the product API (operator on the GPU)."""
    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200.synth import voronoi_scene

    n = c["size"]
    op = product_operator(c)
    truths = np.stack([voronoi_scene(int(s), n) for s in seeds])
    clean = np.asarray(op.apply(truths))
    ys = np.stack([clean[i] + rv.gaussian_noise(clean.shape[1:], c["sigma"], int(s))
                   for i, s in enumerate(seeds)])
    return op, truths, ys


def product_operator(c):
    import paper_1805_02158_b200 as rv

    n = c["size"]
    if c["kind"] == "sr":
        return rv.BlurDownsample(rv.make_psf("gaussian", 7, 1.6), 3, (n, n))
    return rv.Blur(rv.make_psf("uniform", 9), (n, n))


def product_denoiser(c):
    import paper_1805_02158_b200 as rv

    if c["den"] == "patch":  # BASELINE.json configs[2]/[4]: fp32 storage, fp64 accumulation
        return rv.PatchWeighted(weight_dtype=c.get("pw_weights", "float64"))
    return {"gaussian": rv.GaussianFilter, "median": rv.Median3,
            "filterbank": lambda: rv.FilterBank(0)}[c["den"]]()


# ----------------------------------------------------------------------------- CPU side
def _oracle_problem(c, seed):
    from oracle import extras
    from oracle import redve_ref as R
    from paper_1805_02158_b200.synth import voronoi_scene

    n = c["size"]
    truth = voronoi_scene(int(seed), n)
    if c["kind"] == "sr":
        op = R.BlurDecimate(R.psf_taps("gaussian", 7, 1.6), 3, (n, n))
    else:
        op = R.CirculantBlur(R.psf_taps("uniform", 9), (n, n))
    y = R.measure(truth, op, c["sigma"], int(seed))
    den = {"gaussian": R.gaussian_filter, "median": extras.median3, "patch": R.patch_weighted,
           "filterbank": extras.FilterBank(0)}[c["den"]]
    red = R.Red(op, y, c["sigma"], ALPHA, den)
    x0 = op.adjoint(y) if c["kind"] == "sr" else y
    return red, x0


def _oracle_solve(args):
    cfg_id, seed, budget = args
    from oracle import redve_ref as R

    c = CONFIGS[cfg_id]
    red, x0 = _oracle_problem(c, seed)
    step, cost = R.red_problem(red)
    x, tr = R.run_cycling(step, x0, budget, c["ve"], 0, KAPPA, objective=cost)
    return len(tr.iters)


def _single_thread_env():
    """One BLAS thread per process (numpy is already imported, so the pools are
    limited at run time, not by the environment alone)."""
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(cfg_id, n_images, iters_per_solve=BUDGET):
    """Oracle port, 1 core.  Full solves for the 256^2 configs; for the large ones a
    bounded number of fixed-point iterations, scaled to solves/s at the iteration
    count the solve takes (the CG route stops early on an exactly stationary step)."""
    c = CONFIGS[cfg_id]
    ref = reference_available()
    kind = "reference" if ref else "port"
    who = "the unmodified reference (baseline/_ref)" if ref else "oracle/redve_ref.py"
    if c["size"] <= 256:
        t0 = time.perf_counter()
        for i in range(n_images):
            (_ref_solve if ref else _oracle_solve)((cfg_id, i, BUDGET))
        dt = time.perf_counter() - t0
        return {"value": n_images / dt, "unit": "solves/s", "cores": 1, "kind": kind,
                "sample": f"{n_images} full solves (200 iterations) by {who}, 1 thread, {dt:.1f} s"}
    iters = 1 if c["kind"] == "sr" else 3
    if ref:
        dt = _ref_iterations((cfg_id, 0, iters))
    else:
        red, x = _oracle_problem(c, 0)
        t0 = time.perf_counter()
        for _ in range(iters):
            x = red.fp_step(x)
        dt = (time.perf_counter() - t0) / iters
    return {"value": 1.0 / (dt * iters_per_solve), "unit": "solves/s", "cores": 1, "kind": kind,
            "sample": f"{iters} fixed-point iteration(s) of one image by {who}, "
                      f"{dt * 1e3:.0f} ms/iteration, scaled to {iters_per_solve} iterations"}


def cpu_baseline_spatial():
    """configs[4] on the CPU: one fixed-point iteration of the configs[4] problem
    at 1536^2 (same operator, denoiser and CG; a full 8192^2 reference
    iteration takes ~10 minutes on one core), scaled by the pixel ratio to
    8192^2 (every piece is O(N) or O(N log N) per iteration).  The unmodified
    reference when baseline/_ref is installed, else the oracle port at 768^2."""
    if reference_available():
        n = 1536
        _, obj, _, x = _ref_problem(2, 0, size=n)
        t0 = time.perf_counter()
        obj.fp_step(x)
        dt = time.perf_counter() - t0
        scale = (8192 / n) ** 2
        return {"value": 1.0 / (dt * scale), "unit": "iterations/s", "cores": 1,
                "kind": "reference",
                "sample": f"1 fixed-point iteration of a {n}^2 SR problem by the unmodified "
                          f"reference (baseline/_ref), {dt:.1f} s, scaled x{scale:.1f} by "
                          f"pixel count to 8192^2"}
    red, x = _oracle_problem(CONFIGS[2], 0)
    t0 = time.perf_counter()
    red.fp_step(x)
    dt = time.perf_counter() - t0
    scale = (8192 / 768) ** 2
    its_s = 1.0 / (dt * scale)
    return {"value": its_s, "unit": "iterations/s", "cores": 1, "kind": "port",
            "sample": f"1 fixed-point iteration of a 768^2 SR problem by oracle/redve_ref.py "
                      f"({dt:.1f} s), scaled x{scale:.1f} by pixel count to 8192^2"}


REF_PATH = os.path.join(REPO, "baseline", "_ref")


def reference_available() -> bool:
    """The UNMODIFIED reference package, pip-installed into baseline/_ref (git-
    ignored, travels to the GPU box with the repo snapshot)."""
    return os.path.isfile(os.path.join(REF_PATH, "redve", "__init__.py"))


def _ref_problem(cfg_id, seed, size=None):
    """BASELINE.json config through the reference's own public API
    (pkg/src/redve: Blur / BlurDownsample, degrade, RedObjective,
    as_fixed_point_problem), the non-reference denoisers plugged in through its
    callable-denoiser protocol (denoisers.py:1-8)."""
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import redve
    from redve.objective import as_fixed_point_problem
    from scipy import ndimage

    from paper_1805_02158_b200.synth import voronoi_scene

    c = CONFIGS[cfg_id]
    n = size or c["size"]
    truth = voronoi_scene(int(seed), n)
    if c["kind"] == "sr":
        op = redve.BlurDownsample(redve.make_psf("gaussian", 7, 1.6), 3, truth.shape)
    else:
        op = redve.Blur(redve.make_psf("uniform", 9), truth.shape)
    y = redve.degrade(truth, op, c["sigma"], seed=int(seed))
    if c["den"] == "median":  # the 3x3 median a reference user would plug in
        den = lambda x: ndimage.median_filter(x, size=3, mode="wrap")
    elif c["den"] == "filterbank":  # no reference implementation exists
        from oracle import extras

        den = extras.FilterBank(0)
    elif c["den"] == "patch":
        den = redve.PatchWeighted()
    else:
        den = redve.GaussianFilter()
    obj = redve.RedObjective(forward=op, y=y, sigma=c["sigma"], alpha=ALPHA, denoiser=den)
    x0 = op.adjoint(y) if c["kind"] == "sr" else y
    return redve, obj, as_fixed_point_problem(obj), x0


def _ref_solve(args):
    """One full reference solve (solvers.py:388-399) of image `seed`."""
    cfg_id, seed, budget = args
    redve, _, prob, x0 = _ref_problem(cfg_id, seed)
    c = CONFIGS[cfg_id]
    _, tr = redve.solve(prob, x0.ravel(), redve.SolveConfig(
        method="fp-ve", ve_method=c["ve"], m=0, kappa=KAPPA, max_inner_steps=budget))
    return len(tr.records)


def _ref_iterations(args):
    """Seconds per reference fixed-point iteration (objective.py:100-121) of image `seed`."""
    cfg_id, seed, iters = args
    _, obj, _, x = _ref_problem(cfg_id, seed)
    t0 = time.perf_counter()
    for _ in range(iters):
        x = obj.fp_step(x)
    return (time.perf_counter() - t0) / iters


def run_reference(a):
    """The reference's CPU path on the host cores: the unmodified redve from
    baseline/_ref when installed, else the oracle port (oracle/redve_ref.py)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _single_thread_env()
    import multiprocessing as mp

    c = CONFIGS[a.config]
    cores = _host_cores()
    kind = "reference" if reference_available() else "port"
    who = ("unmodified reference redve (baseline/_ref), " if kind == "reference"
           else "oracle/redve_ref.py restatement (baseline/_ref absent), ")
    if a.config == 4:  # one huge image: the CPU path is a single process
        cpu = cpu_baseline_spatial()
        line = {"impl": "reference", "metric": SPATIAL_METRIC, "value": cpu["value"],
                "unit": "iterations/s", "n_gpus": a.gpus, "steps": 1, "warmup": 0,
                "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": c["workload"], "sample": cpu["sample"]},
                "cpu_baseline": cpu,
                "e2e": {"value": cpu["value"], "unit": "iterations/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    solve_fn = _ref_solve if kind == "reference" else _oracle_solve
    nb = a.batch or c["batch"]
    # the native arm's workload at --gpus N: N batches of nb (weak scaling) or
    # one batch of nb split across the ranks (strong); each timed step here
    # solves nb of those images (a bounded sample; the rate is per image)
    global_batch = nb * a.gpus if c["scaling"] == "weak" else nb
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores, initializer=_single_thread_env) as pool:
        if c["size"] <= 256:
            # every timed step solves the whole batch (configs[1]: all 64 images,
            # 200 iterations each); warm-up steps solve one image per worker
            work = [(a.config, i, BUDGET) for i in range(nb)]
            for it in range(a.warmup + a.steps):
                batch = work[:min(cores, nb)] if it < a.warmup else work
                t0 = time.perf_counter()
                pool.map(solve_fn, batch, chunksize=1)
                if it >= a.warmup:
                    times.append(time.perf_counter() - t0)
            ms = 1e3 * statistics.mean(times)
            value = nb / (ms / 1e3)
            sample = (f"{nb} of the {global_batch} images x {BUDGET} iterations per step, "
                      f"process pool of {cores}" if global_batch != nb else
                      f"all {nb} images x {BUDGET} iterations per step, process pool of {cores}")
        else:
            # large images: a bounded sample of fixed-point iterations, one image per
            # core, scaled to solves/s at BUDGET iterations per solve
            iters = 2
            if kind == "reference":
                per = pool.map(_ref_iterations, [(a.config, i, iters) for i in range(cores)],
                               chunksize=1)
            else:
                per = [cpu_baseline(a.config, 1)["value"]]
            t_it = statistics.mean(per) if kind == "reference" else 1.0 / (per[0] * BUDGET)
            value = cores / (t_it * BUDGET)
            ms = None
            sample = (f"{iters} fixed-point iterations of {cores} images (one per core), "
                      f"{t_it * 1e3:.0f} ms/iteration, scaled to {BUDGET} iterations per solve")
    line = {
        "impl": "reference", "metric": METRIC if a.config == 1 else
        f"RED-FP+VE image solves/sec (configs[{a.config}])", "value": value, "unit": "solves/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": c["workload"], "sample": sample,
                                        "global_batch": global_batch},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": kind,
                         "sample": who + sample},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU side
class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region.

    NVML (nvidia-ml-py) is polled from a background thread every 20 ms: a
    cheap query, unlike an ``nvidia-smi -lms`` loop whose start-up and
    per-sample queries measurably stalled short timed regions (configs[0]:
    7.5 -> 10.8 ms per step).  nvidia-smi remains the fallback."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    PERIOD = 0.02

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.window = None
        self.first = ""
        self.thread = None
        self.samples = []  # (time, sm_mhz, [reason names])
        self.smax = None

    def mark(self, t0, t1):
        """Wall-clock bounds of the timed region: only samples inside it count."""
        self.window = (t0, t1)

    def start(self):
        if os.environ.get("REDVE_BENCH_NO_SMI") == "1":  # diagnostics only
            return
        if self._start_nvml():
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        # wait for the first sample: nvidia-smi's start-up must not overlap the timed region
        import select

        ready, _, _ = select.select([self.proc.stdout], [], [], 15.0)
        self.first = self.proc.stdout.readline() if ready else ""

    def _start_nvml(self):
        try:
            import threading

            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                                  None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = [(nv.nvmlClocksThrottleReasonHwSlowdown, "hw_slowdown"),
                    (nv.nvmlClocksThrottleReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                    (nv.nvmlClocksThrottleReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                    (nv.nvmlClocksThrottleReasonSwPowerCap, "sw_power_cap")]
        except Exception:
            return False
        self._stop_evt = threading.Event()

        def poll():
            while not self._stop_evt.is_set():
                try:
                    mhz = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    mem = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM))
                    r = get_reasons(h)
                    self.samples.append((time.time(), mhz, [n for b, n in bits if r & b], mem))
                except Exception:
                    pass
                self._stop_evt.wait(self.PERIOD)

        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        while not self.samples and self.thread.is_alive():
            time.sleep(0.005)
        return True

    def _in_window(self, rows):
        if self.window is None:
            return rows
        lo, hi = self.window[0] - 0.025, self.window[1] + 0.025
        inside = [r for r in rows if r[0] is not None and lo <= r[0] <= hi]
        return inside or rows[-1:]  # a region shorter than the period: the nearest sample

    def _summary(self, rows, smax):
        sm = [r[1] for r in rows if r[1] is not None]
        mem = [r[3] for r in rows if len(r) > 3 and r[3] is not None]
        reasons = sorted({n for r in rows for n in r[2]})
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
               "reasons": reasons, "samples": len(sm)}
        if mem:
            out["mem_mhz"] = statistics.median(mem)
        return out

    def stop(self):
        if self.thread is not None:
            self._stop_evt.set()
            self.thread.join(timeout=5)
            return self._summary(self._in_window(self.samples), self.smax)
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        out = self.first + out
        rows, smax = [], None
        for line in out.strip().splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            try:
                mhz, smax = float(f[1]), float(f[2])
            except ValueError:
                continue
            rows.append((ts, mhz, [n for n, v in zip(self.NAMES, f[5:9])
                                   if v.lower().startswith("active")]))
        return self._summary(self._in_window(rows), smax)


def algorithmic_bytes(kind, B, N, s=8, kp1=KAPPA + 1, npos=24, iters=20, ws=8):
    """Bytes each kernel must move per launch (each logical array read/written once);
    ws = bytes per PatchWeighted raw weight (4 with fp32 planes)."""
    table = {
        "row_fwd": 2 * B * N * s,            # read x, write the pair spectrum
        "col": 2 * B * N * s + N * 8,        # read+write the spectrum, read g
        "row_inv": 4 * B * N * s,            # read spectrum, x_b, x_prev; write x+
        "cost": 3 * B * N * s,               # read x, y, reference
        "copy_view": 2 * B * N * s,
        "gram": (kp1 + 1) * B * N * s,       # kappa+2 window iterates
        "combine": (kp1 + 1) * B * N * s,    # kappa+1 iterates read, 1 written
        "gather": 2 * B * N * s,
        "filter_bank": 2 * B * N * s,        # read x, write f
        "cg_matvec": 4 * B * N * s,          # read r, p_old; write p, q
        "cg_update": 6 * B * N * s,          # read x, p, r, q; write x, r
        # the ALGORITHM's bytes: read x, write f, and the balancing field D read and
        # written once per sweep (weights recomputable from x on chip); the
        # implementation streams 24 stored weight planes per sweep on top
        # (pw_implementation_bytes), which this does not credit
        "patch_weighted": B * N * s * (2 + 2 * iters),
        # spectral route on chip (k_spec_run, one launch per solve): per step the
        # spectrum in / out and the constants m, Xb (complex, 16 B), per cycle
        # the VE window twice (Gram, recombination)
        "spec_run": B * N * 16 * (4 * BUDGET + 2 * (kp1 + 1) * (BUDGET // kp1)),
        # slab primitives of the spatial solve (configs[4])
        "normal_matvec": 2 * B * N * s,      # read w, write out
        "vec_reduce": 2 * B * N * s,         # read x, y
        "vec_axpby": 3 * B * N * s,          # read x, y; write y
        "fidelity": B * N * s + B * N * s // 9,
        "window_gram": (kp1 + 1) * B * N * s,
        "window_combine": (kp1 + 1) * B * N * s,
        "halo_push": 2 * B * N * s,          # read the slab, write it (+ 2 halo strips)
    }
    return table.get(kind)


def pw_implementation_bytes(B, N, s=8, npos=24, iters=20, ws=8):
    """What the PatchWeighted kernels actually stream: raw weights (read x, write
    the 24 half-plane planes), each sweep (read the planes + D, write D), apply
    (read planes, D, x, write f) -- 572 N s with fp64 planes, 308 N s with fp32."""
    return B * N * (s + npos * ws + iters * (npos * ws + 2 * s) + npos * ws + 3 * s)


def _pw_ws(c):
    return 4 if c.get("pw_weights") == "float32" else 8


def algorithmic_flops(kind, B, N, nf=8, fs=5):
    """fp64 flops per launch of the compute-bound kernels (FMA = 2 flops)."""
    if kind == "filter_bank":  # nf correlations + nf adjoint convolutions of fs x fs per pixel
        return B * N * nf * fs * fs * 2 * 2
    return None


def fp64_peak():
    p = os.path.join(REPO, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["fp64_fma_tflops"]), \
                "measured (profiles/fp64_peak.json: tools/fp64_peak.cu FMA chains on this B200 pool)"
    return 37.2, "nominal 148 SMs x 64 FP64 FMA/clk x 1.965 GHz"


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


def ncu_traffic_for(kind, config):
    """Per-launch DRAM traffic of `kind` on `config`: config-keyed entries
    ("patch_weighted:c4": the composite's kernels summed over one call) first,
    the configs[1] kernel table otherwise."""
    v = ncu_traffic(f"{kind}:c{config}")
    if v is None and config == 1:
        v = ncu_traffic(kind)
    return v


def init_ranks(world, local):
    """One rank per GPU over NCCL.  When the node has fewer GPUs than ranks
    (plumbing checks on a 1-GPU box), ranks share devices round-robin and the
    few host-side reductions go over gloo; such a line says "shared_gpus" and
    is not a scaling measurement."""
    import torch
    import torch.distributed as dist

    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    shared = world > ndev
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return shared


def _reduce_max(t, world, shared):
    """Max over ranks of a 1-element device tensor (gloo path via the host)."""
    import torch.distributed as dist

    if world <= 1:
        return float(t.item())
    if shared:
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        return float(h.item())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def settle_solves(solve, tol=0.01, budget_s=4.0):
    """Extra untimed solves after the W warm-up ones until three consecutive solves
    take the same device time (within ``tol``), at most ``budget_s`` seconds.
    On a freshly acquired box the first second of GPU work ran up to 2x slow
    (a first bench on a fresh box after pytest measured 45.6 ms per configs[1]
    step, the same build 20.4 ms on the next run), so the timed region must not
    start inside that transient.  Returns the number of extra solves."""
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hist, n, t0 = [], 0, time.time()
    while time.time() - t0 < budget_s:
        e0.record()
        solve()
        e1.record()
        torch.cuda.synchronize()
        n += 1
        ms = e0.elapsed_time(e1)
        hist.append(ms)
        if len(hist) >= 3 and max(hist[-3:]) - min(hist[-3:]) <= tol * min(hist[-3:]):
            break
    return n


def run_native(a):
    import torch
    import torch.distributed as dist

    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200 import _native as nat
    from paper_1805_02158_b200.shard import shard_bounds

    c = CONFIGS[a.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = init_ranks(world, local)
    local = local % torch.cuda.device_count()
    nb = a.batch or c["batch"]
    if c["scaling"] == "strong":  # a global batch split across the ranks
        lo, hi = shard_bounds(nb, world, rank)
        seeds, global_batch = range(lo, hi), nb
    else:                         # every rank its own batch
        seeds, global_batch = range(rank * nb, rank * nb + nb), nb * world
    B, n = len(seeds), c["size"]
    N = n * n
    op, truths, ys = make_inputs_gpu(c, seeds)
    den = product_denoiser(c)
    cfg = rv.SolveConfig(method="fp-ve", ve_method=c["ve"], m=0, kappa=KAPPA, max_inner_steps=BUDGET)
    y_dev = torch.from_numpy(ys).cuda()
    batch = rv.RedBatch(op, y_dev, c["sigma"], ALPHA, den)
    if c["kind"] == "sr":  # zero-filled adjoint initialisation (cli.py:360-361)
        x0 = torch.from_numpy(np.asarray(op.adjoint(ys))).cuda()
    else:
        x0 = y_dev.clone()

    def barrier():
        if world > 1:
            dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    # warm up exactly as the timed loop runs: the previous result stays alive while
    # the next solve allocates its output (two output buffers in the allocator's
    # cache; otherwise the second timed step pays a 33 MB cudaMalloc, +1.4 ms)
    keep = [None]

    def warm_solve():
        keep[0] = batch.solve(x0, cfg)

    for _ in range(a.warmup):
        warm_solve()
    torch.cuda.synchronize()
    settle = settle_solves(warm_solve)
    res, keep[0] = keep[0], None  # exactly one earlier result alive, as inside the loop

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    l0 = nat.kernel_launches()
    tw0 = time.time()
    e0.record(stream)
    marks = []  # per-step boundaries (diagnostic: a slow step shows up by itself)
    for _ in range(a.steps):
        res = batch.solve(x0, cfg)
        marks.append(torch.cuda.Event(enable_timing=True))
        marks[-1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(tw0, time.time())
    step_ms = [round(p.elapsed_time(q), 3) for p, q in zip([e0] + marks[:-1], marks)]
    l1 = nat.kernel_launches()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / a.steps
    ms = _reduce_max(torch.tensor([ms], dtype=torch.float64, device="cuda"), world, shared)
    value = global_batch / (ms / 1e3)
    launches = (l1 - l0) // a.steps
    assert int((res.status != 0).sum()) == 0
    iters = int(res.n_records.max())

    # ---- the other drivers configs[1] names (FP, FP+RRE), same batch, same timing
    methods = {f"fp-ve/{c['ve']}": {"value": value, "ms_per_step": ms,
                                    "iterations": iters}}
    if a.config == 1:
        for label, mcfg in (("fp", rv.SolveConfig(method="fp", max_inner_steps=BUDGET)),
                            ("fp-ve/rre", rv.SolveConfig(method="fp-ve", ve_method="rre", m=0,
                                                         kappa=KAPPA, max_inner_steps=BUDGET))):
            for _ in range(a.warmup):
                r2 = batch.solve(x0, mcfg)  # result lifetimes as in the timed loop
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(a.steps):
                r2 = batch.solve(x0, mcfg)
            e1.record(stream)
            torch.cuda.synchronize()
            mms = e0.elapsed_time(e1) / a.steps
            mms = _reduce_max(torch.tensor([mms], dtype=torch.float64, device="cuda"), world,
                              shared)
            assert int((r2.status != 0).sum()) == 0
            methods[label] = {"value": global_batch / (mms / 1e3), "ms_per_step": mms,
                              "iterations": int(r2.n_records.max())}

    # ---- per-kernel device times (CUDA events bracketing every launch, one extra solve)
    nat.profile(True)
    batch.solve(x0, cfg)
    rep = nat.profile_report()
    nat.profile(False)
    kernels = {}
    for kind, (tot, cnt) in rep.items():
        ab = algorithmic_bytes(kind, B, N, ws=_pw_ws(c))
        avg = tot / cnt
        kernels[kind] = {"launches": cnt, "avg_us": 1e3 * avg, "total_ms": tot,
                         "gbs": None if ab is None else ab / (avg / 1e3) / 1e9}
        if kind == "patch_weighted":  # what the stored-plane design streams
            kernels[kind]["impl_gbs"] = pw_implementation_bytes(B, N, ws=_pw_ws(c)) / (avg / 1e3) / 1e9
    step_kernel_ms = sum(v["total_ms"] for v in kernels.values())
    dom = max((k for k in kernels if kernels[k]["gbs"] is not None),
              key=lambda k: kernels[k]["total_ms"])
    fl = algorithmic_flops(dom, B, N)
    if fl is not None:  # compute-bound stencil: fp64 FMA roofline
        tfs = fl / (kernels[dom]["avg_us"] * 1e-6) / 1e12
        kernels[dom]["tflops"] = tfs
        peak, peak_src = fp64_peak()
        roof = {"bound": "fp64", "kernel": dom, "achieved": tfs, "peak": peak, "unit": "TFLOP/s",
                "frac": tfs / peak, "peak_source": peak_src,
                "share_of_step": kernels[dom]["total_ms"] / step_kernel_ms,
                "algorithmic_flops_per_launch": fl, "traffic": None}
    else:
        peak, peak_src = measured_peak()
        ach = kernels[dom]["gbs"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": None if ach is None else ach / peak, "peak_source": peak_src,
                "share_of_step": kernels[dom]["total_ms"] / step_kernel_ms,
                "algorithmic_bytes_per_launch": algorithmic_bytes(dom, B, N, ws=_pw_ws(c)),
                "traffic": ncu_traffic_for(dom, a.config)}

    # whole-step roofline against SURVEY.md 8(d)'s per-iteration algorithmic
    # bytes for the deblur step, N s (2 + 7.5 + 2 + 1 + (2k+3)/(m+k+1) + 4/c)
    step_roof = None
    if c["kind"] == "deblur":
        cad = 5 if N > 16384 else 1
        units = 2 + 7.5 + 2 + 1 + (2 * KAPPA + 3) / (0 + KAPPA + 1) + 4 / cad
        bpi = units * B * N * 8
        gbs = bpi / (ms / max(iters, 1) * 1e-3) / 1e9
        hbm = measured_peak()[0]
        step_roof = {"model": "SURVEY.md 8(d): N*s*(2+7.5+2+1+(2k+3)/(m+k+1)+4/c) per image-iteration",
                     "units_per_image_iteration": units, "bytes_per_iteration": bpi,
                     "achieved_gbs": gbs, "peak": hbm, "frac": gbs / hbm}

    # ---- e2e through the public API with host buffers (pinned, allocated up front):
    # problem setup from the host measurements, H2D of y and x0, the solve, D2H of
    # the solutions (traces come back inside solve_batch)
    ys_host = torch.from_numpy(ys).pin_memory()
    # deblurring starts from x0 = y (cli.py:362-363): the user hands the same
    # array, which RedBatch already uploaded; SR starts from the adjoint
    x0_is_y = c["kind"] != "sr"
    x0_host = ys_host if x0_is_y else x0.cpu().pin_memory()
    x_host = torch.empty(x0.shape, dtype=torch.float64).pin_memory()
    e2e_steps = max(1, a.steps)

    def e2e_step(phases=None):
        t_a = time.perf_counter()
        b2 = rv.RedBatch(op, ys_host, c["sigma"], ALPHA, den)
        t_b = time.perf_counter()
        X, trs = rv.solve_batch(b2, x0_host, cfg)
        t_c = time.perf_counter()
        x_host.copy_(X)
        torch.cuda.synchronize()
        if phases is not None:
            phases.append((t_b - t_a, t_c - t_b, time.perf_counter() - t_c))
        del b2
        return trs

    # warm-up as for the device timing: W steps, then until two consecutive
    # steps agree (buffer cache, graph capture, pinned staging, host allocator)
    w_ms = []
    for i in range(a.warmup + 20):
        t_w = time.perf_counter()
        e2e_step()
        w_ms.append(1e3 * (time.perf_counter() - t_w))
        if i + 1 >= a.warmup and len(w_ms) >= 2 and abs(w_ms[-1] - w_ms[-2]) <= 0.05 * w_ms[-2]:
            break
    barrier()
    phases = []
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        traces = e2e_step(phases)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_s = _reduce_max(torch.tensor([e2e_s], dtype=torch.float64, device="cuda"), world, shared)
    assert len(traces) == B
    # ---- the same steps through the pipelined public API (rv.solve_stream): step
    # i+1's H2D and step i-1's D2H ride on a copy stream under step i's kernels.
    # Every step still uploads its measurements and reads its solutions and traces.
    item = ys_host if x0_is_y else (ys_host, x0_host)

    def piped(nsteps):
        n_done = 0
        for xh, trs in rv.solve_stream(op, (item for _ in range(nsteps)), c["sigma"], ALPHA, den,
                                       cfg):
            assert len(trs) == B
            n_done += 1
        return n_done

    piped(max(a.warmup, 3))
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n_piped = piped(e2e_steps)
    torch.cuda.synchronize()
    pipe_s = (time.perf_counter() - t0) / n_piped
    pipe_s = _reduce_max(torch.tensor([pipe_s], dtype=torch.float64, device="cuda"), world, shared)
    serial_s = e2e_s
    e2e_mode = "serial"
    if pipe_s < e2e_s:
        e2e_s, e2e_mode = pipe_s, "pipelined (solve_stream: copies of steps i-1, i+1 under step i)"
    h2d = ys.nbytes + (0 if x0_is_y else x0.numel() * 8)  # measurements (+ x0 for SR)
    d2h = x0.numel() * 8 + B * (BUDGET * 5 * 8)  # solutions + per-record trace arrays

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        _single_thread_env()
        cpu = cpu_baseline(a.config, a.cpu_images if c["size"] <= 256 else 1, iters)

    if rank == 0:
        line = {
            "metric": METRIC if a.config == 1 else f"RED-FP+VE image solves/sec (configs[{a.config}])",
            "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": c["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": c["workload"], "global_batch": global_batch,
                       "images_per_gpu": B, "image": f"{n}x{n}", "iterations": iters,
                       "ms_per_iteration": ms / max(iters, 1), "parallelism": f"dp{world}",
                       **({"shared_gpus": True} if shared else {}),
                       **({"pw_weight_planes": c["pw_weights"]} if "pw_weights" in c else {}),
                       "l2": "working set > L2 (ring of kappa+2 iterates per image)"
                       if B * N * 8 * (KAPPA + 2) > 126e6 else "working set fits L2"},
            "e2e": {"value": global_batch / e2e_s, "unit": "solves/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s, "mode": e2e_mode,
                    "serial": {"value": global_batch / serial_s, "ms_per_step": 1e3 * serial_s},
                    "pipelined": {"value": global_batch / pipe_s, "ms_per_step": 1e3 * pipe_s},
                    "warmup_ms": [round(v, 2) for v in w_ms],
                    "phase_ms": {k: round(1e3 * statistics.median(v), 3) for k, v in
                                 zip(("setup_h2d_y", "solve_h2d_x0_traces", "d2h_x"),
                                     zip(*phases))}},
            "gpu_launches": int(launches),
            "settle_solves": settle,
            "step_ms": step_ms,
            "methods": methods,
            "roofline": roof,
            "step_roofline": step_roof,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_spatial(a):
    """configs[4]: one 8192^2 SR image split into row slabs across the ranks."""
    import torch
    import torch.distributed as dist

    import paper_1805_02158_b200 as rv
    from paper_1805_02158_b200 import _native as nat
    from paper_1805_02158_b200.spatial import PeerComm, SpatialProblem, solve_spatial
    from paper_1805_02158_b200.synth import voronoi_scene

    c = CONFIGS[4]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shared = init_ranks(world, local)
    local = local % torch.cuda.device_count()
    n = c["size"]
    op = product_operator(c)
    truth = voronoi_scene(0, n)
    clean = np.asarray(op.apply(truth))
    y = clean + rv.gaussian_noise(clean.shape, c["sigma"], 0)
    x0 = np.asarray(op.adjoint(y))            # zero-filled adjoint initialisation
    del clean
    den = product_denoiser(c)
    # halos by peer-memory stores; allreduces on gloo (host tensors) when the
    # ranks share one GPU, NCCL otherwise
    comm = PeerComm(device="cpu" if shared else "cuda")
    prob = SpatialProblem(op, y, c["sigma"], ALPHA, den, comm=comm, reference=truth)
    cfg = rv.SolveConfig(method="fp-ve", ve_method="rre", m=0, kappa=KAPPA,
                         max_inner_steps=SPATIAL_BUDGET)
    gather = prob.gather
    x0_slab = prob.slab(x0)                   # resident in HBM before the timed region

    def one_step():
        prob.gather = lambda x, out=None: x  # the timed step keeps the result on the device
        try:
            return solve_spatial(prob, x0_slab, cfg)
        finally:
            prob.gather = gather

    def barrier():
        if world > 1:
            dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(a.warmup):
        one_step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    l0 = nat.kernel_launches()
    tw0 = time.time()
    e0.record(stream)
    for _ in range(a.steps):
        _, tr = one_step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(tw0, time.time())
    l1 = nat.kernel_launches()
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / a.steps
    ms = _reduce_max(torch.tensor([ms], dtype=torch.float64, device="cuda"), world, shared)
    iters = len(tr.records)
    value = iters / (ms / 1e3)

    nat.profile(True)
    one_step()
    rep = nat.profile_report()
    nat.profile(False)
    lay = prob.lay
    kernels = {}
    ext_rows = {"patch_weighted": lay.Hext, "upsample_corr": lay.Hext,
                "normal_matvec": prob.op_lay.Hext}  # extended slabs (denoiser / operator halo)
    for kind, (tot, cnt) in rep.items():
        units = ext_rows[kind] * n if kind in ext_rows else lay.rows * n
        ab = algorithmic_bytes(kind, 1, units, ws=_pw_ws(c))
        avg = tot / cnt
        kernels[kind] = {"launches": cnt, "avg_us": 1e3 * avg, "total_ms": tot,
                         "gbs": None if ab is None else ab / (avg / 1e3) / 1e9}
        if kind == "patch_weighted":  # what the stored-plane design streams
            kernels[kind]["impl_gbs"] = pw_implementation_bytes(1, units, ws=_pw_ws(c)) / (avg / 1e3) / 1e9
    step_kernel_ms = sum(v["total_ms"] for v in kernels.values())
    dom = max((k for k in kernels if kernels[k]["gbs"] is not None),
              key=lambda k: kernels[k]["total_ms"])
    peak, peak_src = measured_peak()
    ach = kernels[dom]["gbs"]
    roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak, "peak_source": peak_src,
            "share_of_step": kernels[dom]["total_ms"] / step_kernel_ms,
            "algorithmic_bytes_per_launch": algorithmic_bytes(
                dom, 1, ext_rows[dom] * n if dom in ext_rows else lay.rows * n, ws=_pw_ws(c)),
            "traffic": ncu_traffic_for(dom, 4)}

    # e2e through the public API: problem setup from the host measurements (H2D of
    # the slab's y and x0), the solve, the gathered host image out.  The timed
    # problem is released first so the new one reuses its device blocks (a user
    # runs one problem of this size at a time).
    del one_step, prob, x0_slab, tr
    import gc

    gc.collect()
    torch.cuda.synchronize()
    barrier()
    # host buffers page-locked up front (the contract's "from pinned host memory");
    # every byte of y, x0, the reference and the result still crosses the bus
    # inside the timed region
    from paper_1805_02158_b200.spatial import PinnedHost

    y_pin, x0_pin, ref_pin = PinnedHost(y), PinnedHost(x0), PinnedHost(truth)
    out_pin = PinnedHost(shape=(n, n))
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    prob2 = SpatialProblem(op, y_pin, c["sigma"], ALPHA, den, comm=comm, reference=ref_pin)
    x_host, _ = solve_spatial(prob2, x0_pin, cfg, out=out_pin)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e_s = _reduce_max(torch.tensor([e2e_s], dtype=torch.float64, device="cuda"), world, shared)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        _single_thread_env()
        cpu = cpu_baseline_spatial()
    if rank == 0:
        line = {
            "metric": SPATIAL_METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": c["workload"], "image": f"{n}x{n}", "iterations": iters,
                       "ms_per_iteration": ms / iters, "parallelism": f"spatial{world}",
                       **({"shared_gpus": True} if shared else {}),
                       "slab_rows": lay.rows, "halo_rows": lay.halo,
                       "pw_weight_planes": c.get("pw_weights", "float64"),
                       "l2": "working set > L2 (8192^2 fp64 = 512 MiB per image)"},
            "e2e": {"value": iters / e2e_s, "unit": "iterations/s",
                    "h2d_bytes_per_step": (sum(1 for g in lay.ext_rows() if g % 3 == 0)
                                           * ((n + 2) // 3) + 2 * lay.rows * n) * 8,
                    "d2h_bytes_per_step": n * n * 8, "ms_per_step": 1e3 * e2e_s},
            "gpu_launches": int((l1 - l0) // a.steps),
            "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        # drop the peer mappings of the neighbours' buffers on every rank before
        # any rank exits (a producer must outlive its IPC consumers)
        del prob2
        gc.collect()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.ipc_collect()  # release what the neighbours have let go of
        barrier()
        dist.destroy_process_group()


def _relaunch_distributed(a) -> bool:
    """``--gpus N`` (N > 1) outside torchrun: start N ranks on this node."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    a = parse()
    _relaunch_distributed(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.impl != "reference" and world != a.gpus:
        print(f"bench: --gpus {a.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}",
              file=sys.stderr)
    if a.impl == "reference":
        run_reference(a)
    elif a.config == 4:
        run_spatial(a)
    else:
        run_native(a)


if __name__ == "__main__":
    main()
