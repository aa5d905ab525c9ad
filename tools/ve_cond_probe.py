"""Device extrapolate_once on the ill-conditioned golden windows vs the
reference: gamma / vector errors per condition number and rule."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1805_02158_b200 as rv

g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "ve_cond.npz"))
for i in range(6):
    rows = g[f"cond{i}/rows"]
    for m in ("mpe", "rre", "svdmpe"):
        res = rv.extrapolate_once(rv.VectorSequenceWindow(rows), m)
        ref = g[f"cond{i}/{m}/vector"]
        gam = g[f"cond{i}/{m}/gamma"]
        spread = np.linalg.norm(np.diff(rows, axis=0))
        ev = np.linalg.norm(np.asarray(res.vector) - ref)
        eg = np.max(np.abs(res.weights.gamma - gam)) / max(np.max(np.abs(gam)), 1e-300)
        print(f"cond {g[f'cond{i}/cond']:.0e} {m:6s} flags {res.converged:d}{res.extrapolated:d}{res.kappa_used} "
              f"gamma rel err {eg:.2e}  |x - ref| {ev:.2e} ( / spread {ev / spread:.2e})", flush=True)
