"""Where does configs[4]'s end-to-end time go (one rank)?  Setup, H2D, solve, gather."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200.spatial import SpatialProblem, TorchComm, solve_spatial
from paper_1805_02158_b200.synth import voronoi_scene

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
op = rv.BlurDownsample(rv.make_psf("gaussian", 7, 1.6), 3, (n, n))
truth = voronoi_scene(0, n)
y = np.asarray(op.apply(truth)) + rv.gaussian_noise(op.out_shape, 5.0, 0)
x0 = np.asarray(op.adjoint(y))
den = rv.PatchWeighted(weight_dtype="float32")
cfg = rv.SolveConfig(method="fp-ve", ve_method="rre", m=0, kappa=5, max_inner_steps=7)
comm = TorchComm(device="cuda")


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(2):
    t0 = tick()
    prob = SpatialProblem(op, y, 5.0, 0.02, den, comm=comm, reference=truth)
    t1 = tick()
    xs = prob.slab(x0)
    t2 = tick()
    g = prob.gather
    prob.gather = lambda x, out=None: x
    xd, tr = solve_spatial(prob, xs, cfg)
    t3 = tick()
    xh = g(xd)
    t4 = tick()
    print(f"setup {1e3 * (t1 - t0):.1f} ms | x0 slab H2D {1e3 * (t2 - t1):.1f} | solve "
          f"{1e3 * (t3 - t2):.1f} | gather D2H {1e3 * (t4 - t3):.1f} | iters {len(tr.records)}")
    del prob, xs, xd, tr
