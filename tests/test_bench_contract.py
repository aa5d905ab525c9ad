"""bench.py's bookkeeping (CPU): the algorithmic byte / flop models DESIGN.md
section 3 states, the config table against BASELINE.json, the unit scaling."""

import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_configs_cover_baseline(bench):
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert sorted(bench.CONFIGS) == list(range(len(base["configs"])))
    for i, c in bench.CONFIGS.items():
        assert c["workload"].startswith(f"configs[{i}]")
    # the super-resolution configs use BASELINE's fp32 storage, everything else fp64
    assert bench._pw_ws(bench.CONFIGS[2]) == 4 and bench._pw_ws(bench.CONFIGS[4]) == 4
    assert bench._pw_ws(bench.CONFIGS[1]) == 8


def test_patch_weighted_bytes(bench):
    N = 1000
    # the algorithm: x in, f out, the balancing field D in + out per sweep (20)
    assert bench.algorithmic_bytes("patch_weighted", 1, N) == 42 * N * 8
    assert bench.algorithmic_bytes("patch_weighted", 3, N, ws=4) == 3 * 42 * N * 8
    # what the kernels stream: (1 + 24 + 20 (24 + 2) + 27) N s with fp64 planes
    assert bench.pw_implementation_bytes(1, N) == 572 * N * 8
    # fp32 planes: N (8 + 24*4 + 20 (24*4 + 16) + 24*4 + 24) = 2464 N = 308 N s
    assert bench.pw_implementation_bytes(1, N, ws=4) == 308 * N * 8


def test_fourier_and_ve_bytes(bench):
    B, N, s = 64, 256 * 256, 8
    assert bench.algorithmic_bytes("row_inv", B, N) == 4 * B * N * s
    assert bench.algorithmic_bytes("row_fwd", B, N) == 2 * B * N * s
    assert bench.algorithmic_bytes("gram", B, N) == 7 * B * N * s     # kappa + 2 iterates
    assert bench.algorithmic_bytes("combine", B, N) == 7 * B * N * s
    assert bench.algorithmic_bytes("no_such_kernel", B, N) is None


def test_filter_bank_flops(bench):
    # 8 filters x 5x5 correlation + adjoint, FMA = 2 flops
    assert bench.algorithmic_flops("filter_bank", 2, 100) == 2 * 100 * 8 * 25 * 2 * 2
    assert bench.algorithmic_flops("row_inv", 2, 100) is None


def test_clock_sampler_keeps_the_timed_window(bench):
    import datetime
    import time

    class FakeProc:
        def __init__(self, out):
            self.out = out

        def terminate(self):
            pass

        def communicate(self, timeout=None):
            return self.out, None

    def stamp(t):
        return datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]

    now = time.time()
    rows = [(now - 1.0, 1200, "Not Active"), (now, 1965, "Active"), (now + 1.0, 1500, "Not Active")]
    out = "\n".join(f"{stamp(t)}, {mhz}, 1965, 500.0, 0x0, Not Active, Not Active, Not Active, {cap}"
                    for t, mhz, cap in rows)
    c = bench.ClockSampler(0)
    c.proc = FakeProc(out)
    c.mark(now - 0.05, now + 0.05)
    got = c.stop()
    assert got["sm_mhz"] == 1965.0 and got["samples"] == 1
    assert got["reasons"] == ["sw_power_cap"]
