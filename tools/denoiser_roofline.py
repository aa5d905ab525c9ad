"""Rooflines of the standalone denoiser / operator kernels at the configs'
shapes (CUDA events around every launch via redve_profile).  Prints one JSON
object; round results are kept in profiles/.

python tools/denoiser_roofline.py > profiles/rNN_denoisers.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200 import _native as nat

HBM = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6539.5
FP64 = json.load(open(os.path.join(os.path.dirname(__file__), "..", "profiles", "fp64_peak.json")))["fp64_fma_tflops"]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    nat.profile(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    rep = nat.profile_report()
    nat.profile(False)
    return {k: (tot / cnt, cnt // reps) for k, (tot, cnt) in rep.items()}


def main():
    g = np.random.default_rng(0)
    out = {"hbm_peak_gbs": HBM, "fp64_peak_tflops": FP64, "kernels": []}

    def add(name, shape, kern, ms, nbytes=None, flops=None):
        e = {"denoiser": name, "shape": shape, "kernel": kern, "ms": ms}
        if nbytes is not None:
            e["gbs"] = nbytes / (ms * 1e-3) / 1e9
            e["frac_hbm"] = e["gbs"] / HBM
            e["algorithmic_bytes"] = nbytes
        if flops is not None:
            e["tflops"] = flops / (ms * 1e-3) / 1e12
            e["frac_fp64"] = e["tflops"] / FP64
        out["kernels"].append(e)

    B, n = 64, 256
    x = torch.from_numpy(g.uniform(0, 255, (B, n, n))).cuda()
    N = B * n * n
    for name, den, kern in (("Median3", rv.Median3(), "median3"),
                            ("GaussianFilter(0.55,5)", rv.GaussianFilter(), "conv")):
        r = timed(lambda: den(x))
        add(name, [B, n, n], kern, r[kern][0], nbytes=2 * N * 8,
            flops=(50 * N if kern == "conv" else None))
    op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
    r = timed(lambda: op.apply(x))
    add("Blur 9x9 apply (operator)", [B, n, n], "conv", r["conv"][0], nbytes=2 * N * 8, flops=162 * N)

    pw = rv.PatchWeighted()
    for m in (768, 4096):
        xs = torch.from_numpy(g.uniform(0, 255, (m, m))).cuda()
        r = timed(lambda: pw(xs), reps=3)
        k, (ms, _) = next(iter(r.items()))
        add("PatchWeighted(1,3,110,20)", [1, m, m], k, ms, nbytes=572 * m * m * 8)

    fb = rv.FilterBank(0)
    xb = torch.from_numpy(g.uniform(0, 255, (128, 512, 512))).cuda()
    r = timed(lambda: fb(xb), reps=3)
    k, (ms, _) = next(iter(r.items()))
    add("FilterBank(8 x 5x5)", [128, 512, 512], k, ms, nbytes=2 * xb.numel() * 8,
        flops=xb.numel() * 8 * 25 * 2 * 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
