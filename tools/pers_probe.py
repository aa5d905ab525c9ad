"""Isolate persistent vs one-shot Fourier-pass differences: one fp_step, and
repeated solves under each setting (determinism)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200.synth import voronoi_scene

SQ = float(np.sqrt(2))
for n, den in ((128, rv.Median3), (256, rv.GaussianFilter)):
    B = 5
    op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
    truths = np.stack([voronoi_scene(s, n) for s in range(B)])
    ys = np.stack([np.asarray(op.apply(truths[i])) + rv.gaussian_noise((n, n), SQ, i) for i in range(B)])
    out = {}
    for flag in ("1", "0", "c", "r"):
        os.environ["REDVE_PERSISTENT"] = flag[0]
        os.environ["REDVE_SPECTRAL"] = "0"
        batch = rv.RedBatch(op, ys, SQ, 0.02, den())
        st, _ = batch.fp_step(ys)
        st = st.cpu().numpy()
        res = batch.solve(ys, rv.SolveConfig(method="fp", max_inner_steps=3))
        out[flag] = (st, res.x.cpu().numpy())
    for a, b in (("1", "0"), ("c", "0"), ("r", "0")):
        d1 = np.abs(out[a][0] - out[b][0]).max()
        d2 = np.abs(out[a][1] - out[b][1]).max()
        print(n, a, b, "fp_step maxdiff", d1, "solve3 maxdiff", d2, flush=True)
