"""Ill-conditioned but full-rank VE windows, extrapolated by the UNMODIFIED
reference (extrapolation.py:319-386), for the Gram-route cutoff question
(csrc/ve.cuh: pivot ratios below max(1e-6, 1e3 rank_tol) go to exact MGS).

    python tests/golden/make_ve_cond_golden.py     (build container only)

Each window has kappa + 2 = 7 iterates of 2048 entries whose difference matrix
U = Q diag(s) V^T has condition number 1e2 ... 1e7, so R's smallest pivot
ratio sweeps across the cutoff.  Writes tests/golden/ve_cond.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from redve import extrapolation as rve  # noqa: E402  (the reference)

CONDS = [1e2, 1e4, 1e5, 3e5, 1e6, 1e7]


def window(cond, seed):
    rng = np.random.default_rng(seed)
    n, k1 = 2048, 6
    q, _ = np.linalg.qr(rng.standard_normal((n, k1)))
    v, _ = np.linalg.qr(rng.standard_normal((k1, k1)))
    s = np.geomspace(1.0, 1.0 / cond, k1) * 50.0
    u = q @ np.diag(s) @ v.T
    x0 = rng.uniform(0, 255, n)
    return np.vstack([x0, x0 + np.cumsum(u.T, axis=0)])


def main():
    out = {}
    for i, c in enumerate(CONDS):
        rows = window(c, 100 + i)
        name = f"cond{i}"
        out[f"{name}/rows"] = rows
        out[f"{name}/cond"] = np.float64(c)
        for method in rve.METHODS:
            res = rve.extrapolate_once(rve.VectorSequenceWindow(rows), method)
            key = f"{name}/{method}"
            out[f"{key}/vector"] = res.vector
            fb = -1 if res.weights is None else int(res.weights.fallback_from is not None)
            out[f"{key}/flags"] = np.array([int(res.converged), int(res.extrapolated),
                                            res.kappa_used, fb], dtype=np.int64)
            if res.weights is not None:
                out[f"{key}/gamma"] = res.weights.gamma
    np.savez_compressed(os.path.join(HERE, "ve_cond.npz"), **out)


if __name__ == "__main__":
    main()
