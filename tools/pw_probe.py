"""Time one PatchWeighted call (and the SR normal operator) at a given size.

python tools/pw_probe.py [n] [reps] [float64|float32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200.spatial import NativeSlabOps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    g = np.random.default_rng(0)
    x = torch.from_numpy(g.uniform(0, 255, (n, n))).cuda()
    wdt = sys.argv[3] if len(sys.argv) > 3 else "float64"
    den = rv.PatchWeighted(weight_dtype=wdt)
    den(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f = den(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    N = n * n
    ws = 4 if wdt == "float32" else 8
    print(f"patch_weighted[{wdt}] {n}x{n}: {ms:.3f} ms/call; 24-plane sweep floor "
          f"{20 * 24 * ws * N / 6.5e12 * 1e3:.2f} ms")
    fwd = rv.BlurDownsample(rv.make_psf("gaussian", 7, 1.6), 3, (n, n))
    ops = NativeSlabOps(fwd, 5.0, 0.02, den)
    ops.normal_matvec(x, 0, n)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        q = ops.normal_matvec(x, 0, n)
    e1.record()
    torch.cuda.synchronize()
    print(f"normal_matvec {n}x{n}: {e0.elapsed_time(e1) / reps:.3f} ms/call "
          f"(2 passes floor {2 * 8 * N / 6.5e12 * 1e3:.3f} ms)")
    for name, fn in (("dot", lambda: ops.dot(x, q)), ("axpby", lambda: ops.axpby(0.5, x, 1.0, q))):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {n}x{n}: {e0.elapsed_time(e1) / reps:.3f} ms/call")


if __name__ == "__main__":
    main()
