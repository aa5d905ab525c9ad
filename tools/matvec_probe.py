"""Time the SR normal operator on one configs[4]-sized slab (8192+2*70 rows x
8192), CUDA events over reps calls; REDVE_MATVEC=generic for the old kernel.
python tools/matvec_probe.py [rows] [cols] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200.spatial import NativeSlabOps

h = int(sys.argv[1]) if len(sys.argv) > 1 else 8192 + 140
w = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
op = rv.BlurDownsample(rv.make_psf("gaussian", 7, 1.6), 3, (8192, 8192))
nat = NativeSlabOps(op, 5.0, 0.02, rv.PatchWeighted())
x = torch.rand((h, w), dtype=torch.float64, device="cuda") * 255
for _ in range(3):
    q = nat.normal_matvec(x, 8192 - 70, 8192)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    q = nat.normal_matvec(x, 8192 - 70, 8192)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / reps * 1e3
gbs = 2 * h * w * 8 / (us * 1e-6) / 1e9
print(f"normal_matvec {h}x{w}: {us:.1f} us/call, {gbs:.0f} GB/s algorithmic (2 N s)")
