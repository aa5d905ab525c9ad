"""Time the filter-bank denoiser on a batch (configs[3] shape by default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_02158_b200 as rv

B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
x = torch.from_numpy(np.random.default_rng(0).uniform(0, 255, (B, n, n))).cuda()
fb = rv.FilterBank(0)
fb(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    fb(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
fl = B * n * n * 8 * (25 * (36 * 36) / 1024 + 25) * 2
print(f"filter_bank {B}x{n}^2: {ms:.3f} ms/call, {fl / ms / 1e9:.1f} TFLOP/s (fp64 FMA count x2)")
