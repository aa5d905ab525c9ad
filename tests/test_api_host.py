"""Host-side API pieces of the drop-in (no GPU): the reference's DFT pair and
PSF embedding helpers (imaging.py:100-130) against the oracle, and the
factor-level VE helpers that are pure host algebra."""

import numpy as np
import pytest

import paper_1805_02158_b200 as rv


def test_dft_pair_and_psf_spectrum_vs_oracle():
    from oracle import redve_ref as R

    x = np.random.default_rng(0).standard_normal((12, 18))
    np.testing.assert_allclose(rv.idft2(rv.dft2(x)), x, atol=1e-12)
    # Parseval with the backward convention
    assert abs(np.sum(x**2) - np.sum(np.abs(rv.dft2(x)) ** 2) / x.size) < 1e-9
    for kind, size, std in (("uniform", 9, None), ("gaussian", 7, 1.6), ("gaussian", 5, 0.55)):
        psf = rv.make_psf(kind, size, std)
        np.testing.assert_allclose(rv.psf_spectrum(psf, (20, 24)),
                                   R.transfer_function(R.psf_taps(kind, size, std), (20, 24)),
                                   atol=1e-13)
        e = rv.embed_psf(psf, (20, 24))
        assert e.sum() == pytest.approx(1.0)
        assert e[0, 0] == psf.taps[psf.radius, psf.radius]
    with pytest.raises(rv.KernelTooLarge):
        rv.embed_psf(rv.make_psf("uniform", 9), (8, 20))
    op = rv.Blur(rv.make_psf("uniform", 9), (20, 24))
    np.testing.assert_allclose(op.spectrum, rv.psf_spectrum(op.psf, (20, 24)))


def test_host_weight_rules():
    from oracle import redve_ref as R

    g = np.random.default_rng(2)
    r = np.triu(g.standard_normal((4, 4))) + 3 * np.eye(4)
    qr = rv.QrFactorization(Q=None, R=r, effective_rank=4, rank_tolerance=1e-12)
    d, gam = R.weights_rre(r)
    np.testing.assert_allclose(rv.gamma_rre(qr).gamma, gam, rtol=1e-12)
    np.testing.assert_allclose(rv.gamma_mpe(qr).gamma, R._annihilate(r, 3)[1], rtol=1e-12)
    xi, eta = rv.reconstruction_coefficients(gam, r)
    np.testing.assert_allclose(xi, 1.0 - np.cumsum(gam[:3]))
    with pytest.raises(rv.RankDeficient):
        rv.gamma_rre(rv.QrFactorization(Q=None, R=r, effective_rank=3, rank_tolerance=1e-12))
    u, s, vt = rv.small_svd(r)
    np.testing.assert_allclose(u @ np.diag(s) @ vt, r, atol=1e-12)
