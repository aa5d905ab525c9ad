"""Factor-level vector-extrapolation API (extrapolation.py:154-316 of the
reference): difference matrix, device MGS QR, weight rules, reconstruction --
against the oracle and the reference's own contracts (orthonormality, QR = U,
weights summing to one, reconstruction = weighted iterate average)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _window(seed=0, k=5, n=4000, decay=0.7):
    g = np.random.default_rng(seed)
    base = g.standard_normal(n)
    rows = [base * decay**j + 1e-2 * g.standard_normal(n) for j in range(k + 2)]
    return np.stack(rows)


def test_difference_matrix_and_qr_contracts():
    import paper_1805_02158_b200 as rv
    from oracle import redve_ref as R

    rows = _window()
    w = rv.VectorSequenceWindow(rows)
    u = rv.build_difference_matrix(w).cpu().numpy()
    np.testing.assert_allclose(u, np.diff(rows, axis=0).T, rtol=0, atol=1e-15)
    qr = rv.mgs_qr(u)
    q = qr.Q.cpu().numpy()
    k = u.shape[1]
    assert qr.effective_rank == k
    np.testing.assert_allclose(q.T @ q, np.eye(k), atol=1e-10)          # orthonormal
    np.testing.assert_allclose(q @ qr.R, u, atol=1e-10 * np.abs(u).max())  # Q R = U
    qo, ro, rank = R.mgs(u)
    assert rank == qr.effective_rank
    np.testing.assert_allclose(qr.R, ro, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("rule", ["mpe", "rre", "svdmpe"])
def test_weight_rules_and_reconstruction(rule):
    import paper_1805_02158_b200 as rv
    from oracle import redve_ref as R

    rows = _window(seed=3)
    w = rv.VectorSequenceWindow(rows)
    qr = rv.mgs_qr(rv.build_difference_matrix(w))
    wt = {"mpe": rv.gamma_mpe, "rre": rv.gamma_rre, "svdmpe": rv.gamma_svdmpe}[rule](qr)
    assert wt.method == rule
    assert abs(wt.gamma.sum() - 1.0) < 1e-12
    x = rv.reconstruct(w, qr, wt)
    np.testing.assert_allclose(x, wt.gamma @ rows[: len(wt.gamma)], rtol=1e-10, atol=1e-10)
    ref = R.extrapolate(rows, rule)
    np.testing.assert_allclose(wt.gamma, ref["gamma"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(x, ref["vector"], rtol=1e-9, atol=1e-9)
    xi, eta = rv.reconstruction_coefficients(wt.gamma, qr.R)
    np.testing.assert_allclose(xi, 1.0 - np.cumsum(wt.gamma[:-1]))
    np.testing.assert_allclose(eta, qr.R[:-1, :-1] @ xi)


def test_error_cases():
    import paper_1805_02158_b200 as rv

    n = 500
    g = np.random.default_rng(1)
    base = g.standard_normal(n)
    with pytest.raises(rv.ZeroFirstColumn):
        rv.mgs_qr(np.zeros((n, 3)))
    # rank-deficient: third difference equals the first
    d = g.standard_normal((n, 2))
    u = np.column_stack([d[:, 0], d[:, 1], d[:, 0]])
    qr = rv.mgs_qr(u)
    assert qr.effective_rank == 2
    with pytest.raises(rv.RankDeficient):
        rv.gamma_rre(qr)
    with pytest.raises(ValueError):
        rv.mgs_qr(u, rank_tolerance=0.0)
    # MPE degenerate sum: differences constructed so that sum(c) = 0
    x0 = base
    rows = np.stack([x0, x0 + base, x0, x0 + base])  # u = [b, -b, b]: dependent
    qr2 = rv.mgs_qr(np.diff(rows, axis=0).T)
    assert qr2.effective_rank == 1
    with pytest.raises(ValueError):
        rv.small_svd(np.zeros((2, 3)))


# ------------------------------------------------ ill-conditioned full-rank windows
@pytest.mark.parametrize("i", range(6))
@pytest.mark.parametrize("method", ["mpe", "rre", "svdmpe"])
def test_ill_conditioned_windows_vs_reference(golden, i, method):
    """Windows with cond(U) = 1e2 ... 1e7 (tests/golden/make_ve_cond_golden.py,
    the unmodified reference's extrapolate_once): R's smallest pivot ratio runs
    from 1e-1 down to 1.3e-6, just above the Gram route's MGS cutoff (1e-6).
    Cholesky of G = U^T U puts ~eps cond^2 on the small pivots, so the weights
    drift from the reference's twice-orthogonalised MGS as cond grows
    (measured: 1e-9 at 1e5, 1.5e-6 at 1e7); the extrapolated point stays within
    1e-7 of the window's own spread, far below the solves' 1e-5 bar."""
    import paper_1805_02158_b200 as rv

    g = golden("ve_cond.npz")
    rows = g[f"cond{i}/rows"]
    cond = float(g[f"cond{i}/cond"])
    key = f"cond{i}/{method}"
    res = rv.extrapolate_once(rv.VectorSequenceWindow(rows), method)
    flags = g[f"{key}/flags"]
    assert (int(res.converged), int(res.extrapolated), res.kappa_used) == tuple(flags[:3])
    assert int(res.weights.fallback_from is not None) == flags[3]
    gam = g[f"{key}/gamma"]
    tol = max(1e-12, 1e-16 * cond**2) * 10
    assert np.max(np.abs(res.weights.gamma - gam)) <= tol * np.max(np.abs(gam)) + 1e-13
    spread = np.linalg.norm(np.diff(rows, axis=0))
    assert np.linalg.norm(np.asarray(res.vector) - g[f"{key}/vector"]) <= 1e-7 * spread
