"""Where does the e2e time go?  configs[1] shapes: problem setup, first solve
(graph capture + instantiate), cached solve, readback."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200.synth import voronoi_scene

B, n = 64, 256
op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
truths = np.stack([voronoi_scene(s, n) for s in range(B)])
ys = np.asarray(op.apply(truths)) + np.stack([rv.gaussian_noise((n, n), 2 ** 0.5, s) for s in range(B)])
cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", max_inner_steps=200)
ysh = torch.from_numpy(ys).pin_memory()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = rv.RedBatch(op, ysh, 2 ** 0.5, 0.02, rv.Median3())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = b.solve(ysh, cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res2 = b.solve(ysh, cfg)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    X, tr = rv.solve_batch(b, ysh, cfg)
    x = X.cpu()
    t4 = time.perf_counter()
    print(f"setup {1e3 * (t1 - t0):.2f} ms | first solve {1e3 * (t2 - t1):.2f} | cached solve "
          f"{1e3 * (t3 - t2):.2f} | solve_batch+D2H {1e3 * (t4 - t3):.2f}")
    del b
