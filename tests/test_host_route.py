"""Host-side logic without a GPU: trace CSV wire format and the caller's-step
drivers (fp / sd / nesterov) of ``solvers.py``.

* CSV: the reference's committed demo traces (pkg/demos/out/deblur_*.csv,
  written by cli.write_trace_csv, cli.py:281-298) are parsed into
  TraceRecords and written back by ``trace_io.write_trace_csv``; the bytes
  must be identical.
* Drivers: a LinearFixedPointProblem and a quadratic with a gradient run
  through ``solve`` against the oracle restatement (oracle/redve_ref.py run_fp,
  solvers.py:288-298) and a direct transcription of the Nesterov recurrence
  (solvers.py:315-337): identical traces and iterates.  The cycling route
  needs the device extrapolation and is covered by the GPU tests.
"""

import numpy as np
import pytest

from paper_1805_02158_b200 import solvers as S
from paper_1805_02158_b200 import trace_io


def _records_from_csv(raw: bytes):
    rows = raw.decode("ascii").strip().splitlines()
    assert rows[0] == "iter,cost,psnr,step_norm,gamma_abs_sum,elapsed_s"
    num = lambda s: None if s == "" else float(s)
    out = []
    for line in rows[1:]:
        it, c, p, sn, g, el = line.split(",")
        out.append(S.TraceRecord(int(it), num(c), num(p), float(sn), num(g), float(el)))
    return out


@pytest.mark.parametrize("name", ["fp", "fp-mpe", "sd", "nesterov"])
def test_trace_csv_bytes_match_reference(golden, tmp_path, name):
    raw = golden("demo64.npz")[f"{name}/csv_bytes"].tobytes()
    tr = S.IterationTrace(records=_records_from_csv(raw))
    path = tmp_path / f"{name}.csv"
    trace_io.write_trace_csv(path, tr)
    assert path.read_bytes() == raw


def test_trace_csv_empty_refused(tmp_path):
    with pytest.raises(ValueError):
        trace_io.write_trace_csv(tmp_path / "x.csv", S.IterationTrace())


def _linear(n=12, seed=0):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = q @ np.diag(np.linspace(-0.6, 0.9, n)) @ q.T
    return S.LinearFixedPointProblem(A=a, b=rng.standard_normal(n))


@pytest.mark.parametrize("tol,budget", [(0.0, 40), (1e-6, 500)])
def test_host_fixed_point_vs_oracle(tol, budget):
    from oracle import redve_ref as R

    lin = _linear()
    prob = lin.problem()
    prob.objective = lambda v: float(v @ v)
    prob.reference = lin.solve()
    x0 = np.ones(12)
    x, tr = S.solve(prob, x0, S.SolveConfig(method="fp", max_inner_steps=budget, tol=tol))
    xo, tro = R.run_fp(lin.step, x0, budget, tol=tol, objective=prob.objective,
                       reference=prob.reference)
    np.testing.assert_array_equal(x, xo)
    a = tro.as_arrays()
    np.testing.assert_array_equal(tr.step_norms(), a["step_norm"])
    np.testing.assert_array_equal(tr.costs(), a["cost"])
    assert tr.inner_steps == len(tro.iters)


def _quadratic(n=10, seed=1):
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((n, n))
    h = m @ m.T / n + np.eye(n)
    c = rng.standard_normal(n)
    return h, c


def test_host_steepest_descent_is_fixed_point_of_gradient_map():
    h, c = _quadratic()
    grad = lambda x: h @ x - c
    prob = S.FixedPointProblem(dimension=10, step=lambda x: x, gradient=grad,
                               objective=lambda x: 0.5 * x @ h @ x - c @ x)
    s = 0.5 / np.linalg.norm(h, 2)
    x, tr = S.run_steepest_descent(prob, np.zeros(10), S.SolveConfig(method="sd", step_size=s,
                                                                      max_inner_steps=30))
    ref = np.zeros(10)
    for _ in range(30):
        ref = ref - s * grad(ref)
    np.testing.assert_array_equal(x, ref)
    assert tr.inner_steps == 30


def test_host_nesterov_recurrence():
    h, c = _quadratic()
    grad = lambda x: h @ x - c
    prob = S.FixedPointProblem(dimension=10, step=lambda x: x, gradient=grad)
    s = 0.9 / np.linalg.norm(h, 2)
    x, tr = S.run_nesterov(prob, np.zeros(10), S.SolveConfig(method="nesterov", step_size=s,
                                                              max_inner_steps=25))
    xr, yr, t = np.zeros(10), np.zeros(10), 1.0
    norms = []
    for _ in range(25):
        xn = yr - s * grad(yr)
        norms.append(np.linalg.norm(xn - xr) / (np.linalg.norm(xr) or 1.0))
        tn = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
        yr = xn + ((t - 1.0) / tn) * (xn - xr)
        xr, t = xn, tn
    np.testing.assert_array_equal(x, xr)
    np.testing.assert_array_equal(tr.step_norms(), norms)


@pytest.mark.parametrize("cfg,msg", [
    (dict(method="sd"), "positive step_size"),
    (dict(method="nesterov"), "positive step_size"),
    (dict(method="sd", step_size=-1.0), "positive step_size"),
])
def test_gradient_methods_validate(cfg, msg):
    prob = S.FixedPointProblem(dimension=3, step=lambda x: x, gradient=lambda x: x)
    with pytest.raises(ValueError, match=msg):
        S.solve(prob, np.ones(3), S.SolveConfig(**cfg))


def test_missing_gradient():
    prob = S.FixedPointProblem(dimension=3, step=lambda x: x)
    with pytest.raises(ValueError, match="needs a gradient"):
        S.solve(prob, np.ones(3), S.SolveConfig(method="sd", step_size=0.1))
    with pytest.raises(ValueError, match="nesterov needs a gradient"):
        S.solve(prob, np.ones(3), S.SolveConfig(method="nesterov", step_size=0.1))


@pytest.mark.parametrize("kw", [dict(method="bogus"), dict(ve_method="x"), dict(kappa=0),
                                dict(m=-1), dict(max_inner_steps=0), dict(tol=-1.0),
                                dict(stabilization_iters=-1),
                                dict(method="fp-ve", max_inner_steps=6)])
def test_solve_config_validation(kw):
    with pytest.raises(ValueError):
        S.SolveConfig(**kw)


def test_nonfinite_iterate_carries_trace():
    prob = S.FixedPointProblem(dimension=2, step=lambda x: x * 1e300)
    with pytest.raises(S.NonFiniteIterate) as ei:
        S.solve(prob, np.ones(2), S.SolveConfig(max_inner_steps=10))
    assert ei.value.trace.inner_steps == 2


def test_x0_checks():
    prob = S.FixedPointProblem(dimension=3, step=lambda x: x)
    with pytest.raises(ValueError, match="dimension"):
        S.solve(prob, np.ones(4), S.SolveConfig())
    with pytest.raises(ValueError, match="non-finite"):
        S.solve(prob, np.array([1.0, np.inf, 0.0]), S.SolveConfig())
