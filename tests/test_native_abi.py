"""CPU-side checks of the C ABI library: it loads, and exports exactly what
include/redve_b200.h declares.  No compute calls (no GPU here)."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "redve_b200.h")
LIB = os.path.join(REPO, "paper_1805_02158_b200", "libredve_b200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(redve_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("redve_create", "redve_denoise", "redve_operator_apply", "redve_problem_create",
                 "redve_fp_step", "redve_cost", "redve_solve", "redve_extrapolate"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.redve_version  # callable without a GPU
    lib.redve_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.redve_version()


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_python_binding_matches_header():
    from paper_1805_02158_b200 import _native

    assert sorted(_native.SYMBOLS) == declared_functions()
    _native.library()


def test_solve_config_validation():
    from paper_1805_02158_b200 import SolveConfig

    with pytest.raises(ValueError):
        SolveConfig(method="bogus")
    with pytest.raises(ValueError):
        SolveConfig(method="fp-ve", kappa=5, max_inner_steps=6)
    with pytest.raises(ValueError):
        SolveConfig(ve_method="xyz")
    SolveConfig(method="fp-ve", kappa=5, max_inner_steps=7)


def test_psf_and_errors_without_gpu():
    import numpy as np

    from paper_1805_02158_b200 import InvalidSize, KernelTooLarge, make_psf
    from paper_1805_02158_b200.imaging import Blur

    assert make_psf("uniform", 9).taps.shape == (9, 9)
    assert abs(make_psf("gaussian", 7, 1.6).taps.sum() - 1.0) < 1e-14
    with pytest.raises(InvalidSize):
        make_psf("uniform", 4)
    with pytest.raises(KernelTooLarge):
        Blur(make_psf("uniform", 9), (8, 8))
    assert np.isfinite(make_psf("gaussian", 5, 0.55).taps).all()
