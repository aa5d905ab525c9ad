"""Solve-by-solve device and wall time of repeated configs[1] solves on one
RedBatch, keeping every result alive (the bench's timed-loop pattern), with
the graph capture counter after each.  python tools/repeat_probe.py [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200 import _native as nat
from paper_1805_02158_b200.synth import voronoi_scene

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
B, n = 64, 256
op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
truths = np.stack([voronoi_scene(s, n) for s in range(B)])
clean = np.asarray(op.apply(truths))
ys = np.stack([clean[i] + rv.gaussian_noise((n, n), float(np.sqrt(2)), i) for i in range(B)])
yd = torch.from_numpy(ys).cuda()
batch = rv.RedBatch(op, yd, float(np.sqrt(2)), 0.02, rv.Median3())
for method, ve in (("fp-ve", "mpe"), ("fp", "mpe"), ("fp-ve", "rre"), ("fp-ve", "mpe")):
    cfg = rv.SolveConfig(method=method, ve_method=ve, m=0, kappa=5, max_inner_steps=200)
    rows = []
    keep = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        res = batch.solve(yd, cfg)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        keep.append(res)
        rows.append({"dev_ms": round(e0.elapsed_time(e1), 2), "call_ms": round(1e3 * (t1 - t0), 2),
                     "wall_ms": round(1e3 * (t2 - t0), 2),
                     "captures": int(batch.graph_captures)})
    print(json.dumps({"method": method, "ve": ve, "rows": rows}), flush=True)
