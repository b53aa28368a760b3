"""GPU path against the committed oracle fixtures (tests/golden/*.json, made
by tests/golden/make_golden.py) at BASELINE sizes: C1 (10^4, both sketches),
the C3-shaped recycling sequence, and C2 (128^3, the bench workload), where
rerunning the CPU oracle would take minutes. Iteration counts within ±2%
(SURVEY.md §8c), status/cycles equal, true residual below tol."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(HERE, f"{name}_oracle.json")) as fh:
        return json.load(fh)


def close_iters(got, want, frac=0.02):
    return abs(got - want) <= max(1, frac * want)


def check_report(rep, g, tol):
    assert rep.status == g["status"]
    assert close_iters(rep.iterations, g["iterations"]), (rep.iterations, g["iterations"])
    assert rep.rhs_norm == pytest.approx(g["rhs_norm"], rel=1e-12)
    if g["status"] == "converged":
        assert rep.final_relative_residual <= tol * (1 + 1e-10)


def test_c1_golden(sk, O):
    g_all = load("c1")
    off, col, val = sk.gen_convdiff(100, -50.0)
    A = sk.SparseMatrix(10000, 10000, off, col, -val)
    b = O.gaussian_vector(10000, 0)
    b /= np.linalg.norm(b)
    for name, g in g_all.items():
        c = g["config"]
        cfg = sk.SolverConfig(m=c["m"], k=c["k"], t=c["t"], s=c["s"], tol=c["tol"], max_restarts=c["max_restarts"])
        S = None if name == "srdct" else sk.SketchOperator.sparse_sign(10000, 120, 0x5EED, 8)
        res = sk.solve(A, b, cfg, sketch=S)
        check_report(res.report, g, c["tol"])
        assert res.report.cycles == g["cycles"]
        # exact counters when the iteration counts agree (counters.hpp books)
        if res.report.iterations == g["iterations"]:
            assert res.report.counters == g["counters"]
            np.testing.assert_allclose(res.x[:16], g["x_head"], rtol=1e-6, atol=1e-9 * g["x_norm"])


def test_c3_small_sequence_golden(sk, O):
    gs = load("c3_small")
    n, count = 64, 5
    b0 = O.gaussian_vector(n * n, 0x3000)
    probs = []
    for i in range(count):
        rel = 1e-3 * (2.0 * O.uniform_stream(0x3100 + i, n * n) - 1.0)
        off, col, val = sk.gen_convdiff2d(n, 100.0 + 2 * i, 100.0 - 2 * i, 0.01 * i, rel)
        A = sk.SparseMatrix(n * n, n * n, off, col, val)
        b = b0 + 0.05 * O.gaussian_vector(n * n, 0x3000 + i) if i else b0.copy()
        probs.append(sk.ProblemInstance(A, b))
    cfg = sk.SolverConfig(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact", max_restarts=20)
    out = sk.solve_sequence(probs, cfg)
    for rep, g in zip(out.reports, gs):
        check_report(rep, g, 1e-8)
    # whole-sequence total (the C3 metric's numerator) within ±2% of the oracle's
    assert close_iters(sum(r.iterations for r in out.reports), sum(g["iterations"] for g in gs))


@pytest.mark.parametrize("device_gen", [True, False])
def test_c2_golden(sk, O, device_gen):
    """The bench workload: 128^3 convection-diffusion, m=100 k=20 t=2 s=240.
    device_gen: operator built on the device (SELL-DIA generator) vs from the
    host CSR (sdr_csr_create, banded detection)."""
    g = load("c2")
    n = g["config"]["n"]
    if device_gen:
        A = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0)
    else:
        off, col, val = sk.gen_convdiff3d(n, 100.0, 50.0, 25.0)
        A = sk.SparseMatrix(n ** 3, n ** 3, off, col, val)
    b = sk.gaussian_vector(n ** 3, 1)
    cfg = sk.SolverConfig(m=100, k=20, t=2, s=240, tol=1e-8)
    res = sk.solve(A, b, cfg)
    check_report(res.report, g, 1e-8)
    assert res.report.cycles == g["cycles"]
    # the true residuals at each restart follow the oracle's
    for (i1, r1), (i2, r2) in zip(res.report.true_residuals, g["true_residuals"]):
        assert i1 == i2
        assert r1 == pytest.approx(r2, rel=1e-3)
    assert np.linalg.norm(res.x) == pytest.approx(g["x_norm"], rel=1e-6)


def _c3_system(sk, i, n=1024):
    N = n * n
    b0 = sk.gaussian_vector(N, 0x3000)
    rel = 1e-3 * (2.0 * sk.uniform_stream(0x3100 + i, N) - 1.0)
    off, col, val = sk.gen_convdiff2d(n, 100.0 + 2 * i, 100.0 - 2 * i, 0.01 * i, rel)
    A = sk.SparseMatrix(N, N, off, col, val)
    b = b0 + 0.05 * sk.gaussian_vector(N, 0x3000 + i) if i else b0
    return A, b


def test_c3_first_system_golden(sk, O):
    """BASELINE C3 at full size (N = 1024^2), first system against the oracle
    run (tests/golden/make_golden.py c3_first)."""
    g = load("c3_first")
    A, b = _c3_system(sk, 0)
    c = g["config"]
    res = sk.solve(A, b, sk.SolverConfig(m=c["m"], k=c["k"], t=c["t"], s=c["s"], tol=c["tol"], variant=c["variant"]))
    assert res.report.status == g["status"]
    assert close_iters(res.report.iterations, g["iterations"])
    assert res.report.cycles == g["cycles"]
    assert res.report.final_relative_residual == pytest.approx(g["final_relative_residual"], rel=1e-6)
    for (i1, r1), (i2, r2) in zip(res.report.true_residuals, g["true_residuals"]):
        assert i1 == i2 and r1 == pytest.approx(r2, rel=1e-6)


def test_c3_sequence_head_with_exact_refresh(sk):
    """The first four systems of the C3 sequence: every system reports a valid status, the
    first matches the standalone first solve, and each matrix change costs k
    matvecs + k sketches of exact refresh (counters, recycle.hpp:297-318)."""
    probs = [sk.ProblemInstance(*_c3_system(sk, i)) for i in range(4)]
    cfg = sk.SolverConfig(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact")
    out = sk.solve_sequence(probs, cfg)
    first = sk.solve(probs[0].matrix, probs[0].rhs, cfg)
    assert out.reports[0].iterations == first.report.iterations
    for r in out.reports:
        assert r.status in ("converged", "max_restarts", "diverged", "breakdown")
        assert r.iterations > 0
    # an exact refresh of the q recycle columns on each change costs q matvecs
    # and q sketches on top of the per-step / per-check / per-cycle counts
    for r in out.reports[1:]:
        extra_mv = r.counters["matvecs"] - r.iterations - len(r.true_residuals)
        extra_sk = r.counters["sketch_applies"] - r.iterations - r.cycles
        assert 1 <= extra_mv <= 21 and extra_mv == extra_sk
