"""The compile-time SR normal operator (k_cg_matvec_ct, csrc/sr.cu: 7 x 7 PSF,
factor 3) against the runtime-(k, s) kernel (REDVE_MATVEC=generic) and the CPU
stand-in, on multi-tile slabs whose global lattice crosses the periodic seam
(heights not divisible by 3, slabs starting off the lattice).

A general PSF takes the same terms in the same order as the generic kernel, so
q = (H^T H / sigma^2 + alpha I) w agrees bit for bit.  A rank-one PSF (the
Gaussian of configs[2]/[4]) is contracted as two 1-D passes in lattice-regular
tiles: the same terms regrouped, equal to rounding."""

import numpy as np
import pytest

from test_spatial_gloo import ALPHA, FACTOR, SIGMA, _Fwd

pytestmark = pytest.mark.gpu

SHAPES = [(200, 300, 0, 200), (157, 131, 0, 157), (97, 193, 5, 8192), (130, 257, 8150, 8192),
          (64, 64, 62, 64), (301, 95, 1, 301)]


def _ops(taps):
    from oracle import extras
    from paper_1805_02158_b200 import Median3
    from paper_1805_02158_b200.spatial import NativeSlabOps
    from spatial_cpu_ops import CpuSlabOps

    nat = NativeSlabOps(_Fwd(taps, FACTOR, (60, 47)), SIGMA, ALPHA, Median3())
    cpu = CpuSlabOps(taps, FACTOR, SIGMA, ALPHA, extras.median3)
    return nat, cpu


def _psf(kind):
    from oracle import redve_ref as R

    if kind == "gaussian":
        return R.psf_taps("gaussian", 7, 1.6)
    t = np.random.default_rng(11).uniform(0.0, 1.0, (7, 7))  # rank 7
    return t / t.sum()


@pytest.mark.parametrize("kind", ["gaussian", "general"])
@pytest.mark.parametrize("h,w,row0,Hg", SHAPES)
def test_ct_vs_generic_and_cpu(monkeypatch, kind, h, w, row0, Hg):
    nat, cpu = _ops(_psf(kind))
    x = np.random.default_rng(h * w + row0).uniform(0, 255, (h, w))
    got = nat.host(nat.normal_matvec(nat.tensor(x), row0, Hg))
    monkeypatch.setenv("REDVE_MATVEC", "generic")
    gen = nat.host(nat.normal_matvec(nat.tensor(x), row0, Hg))
    if kind == "general":
        np.testing.assert_array_equal(got, gen)
    else:
        assert np.abs(got - gen).max() <= 1e-13 * np.abs(gen).max()
    want = cpu.host(cpu.normal_matvec(cpu.tensor(x), row0, Hg))
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
