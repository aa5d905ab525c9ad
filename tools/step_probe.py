"""Per-kernel device times of one configs[1] solve (or a configs[0]/[3] shape),
plus the graph-replayed solve time.  Experiment loop for the Fourier kernels.

python tools/step_probe.py [B] [n] [method] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200 import _native as nat
from paper_1805_02158_b200.synth import voronoi_scene

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
method = sys.argv[3] if len(sys.argv) > 3 else "fp-ve"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
den = os.environ.get("PROBE_DEN", "median")
op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
truths = np.stack([voronoi_scene(s, n) for s in range(B)])
clean = np.asarray(op.apply(truths))
ys = np.stack([clean[i] + rv.gaussian_noise((n, n), float(np.sqrt(2)), i) for i in range(B)])
cfg = rv.SolveConfig(method=method, ve_method="mpe", m=0, kappa=5, max_inner_steps=200)
yd = torch.from_numpy(ys).cuda()
dn = {"median": rv.Median3, "gaussian": rv.GaussianFilter, "fb": lambda: rv.FilterBank(0)}[den]()
batch = rv.RedBatch(op, yd, float(np.sqrt(2)), 0.02, dn)
for _ in range(3):
    res = batch.solve(yd, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    res = batch.solve(yd, cfg)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
nat.profile(True)
batch.solve(yd, cfg)
rep = nat.profile_report()
nat.profile(False)
out = {"B": B, "n": n, "method": method, "den": den, "ms_per_solve": ms,
       "solves_per_s": B / ms * 1e3,
       "kernels_us": {k: round(1e3 * t / c, 2) for k, (t, c) in rep.items()},
       "kernels_ms_total": {k: round(t, 3) for k, (t, c) in rep.items()}}
print(json.dumps(out))
