"""Trace comparison against reference fixtures, shared by the GPU parity tests.

A reference trace (solvers.py:51-95) is matched record by record: identical
record count, costs to ``cost_rtol``, PSNR within 0.01 dB (north_star), step
norms to ``sn_rtol`` above fp64 rounding (``sn_atol``), and the accepted
extrapolations (records carrying gamma_abs_sum) wherever the reference's step
norm is above ``sig_floor``.  Below that floor the reference extrapolates fp64
rounding noise: its weights are noise, and the spectral route's iterates are
exactly stationary there (csrc/spectral.cuh), so only the signal regime is
compared.
"""

import numpy as np


def _opt(v):
    return np.nan if v is None else v


def cmp_trace(tr, g, key, cost_rtol=1e-9, sn_rtol=1e-6, sn_atol=1e-13, sig_floor=1e-12):
    np.testing.assert_array_equal(np.array([r.iter for r in tr.records]), g[f"{key}/iter"])
    cost, gc = tr.costs(), g[f"{key}/cost"]
    assert np.array_equal(np.isnan(cost), np.isnan(gc))
    m = ~np.isnan(gc)
    np.testing.assert_allclose(cost[m], gc[m], rtol=cost_rtol)
    ps = np.array([_opt(r.psnr) for r in tr.records])
    gp = g[f"{key}/psnr"]
    assert np.array_equal(np.isnan(ps), np.isnan(gp))
    m = ~np.isnan(gp)
    assert np.max(np.abs(ps[m] - gp[m]), initial=0.0) <= 0.01
    sn, gs = tr.step_norms(), g[f"{key}/step_norm"]
    np.testing.assert_allclose(sn, gs, rtol=sn_rtol, atol=sn_atol)
    gam = np.array([_opt(r.gamma_abs_sum) for r in tr.records])
    gg = g[f"{key}/gamma_abs_sum"]
    sig = gs > sig_floor
    assert np.array_equal(np.isnan(gam)[sig], np.isnan(gg)[sig])
    n_sig = int(np.sum(~np.isnan(gg) & sig))
    assert n_sig <= len(tr.cycle_weights) <= int(g[f"{key}/n_cycles"])
