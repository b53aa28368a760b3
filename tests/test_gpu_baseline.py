"""Device classical restarted GMRES (baseline.hpp:51-216)
against the oracle restatement (oracle/skrylov_oracle.hpp baseline_gmres):
statuses, iteration counts, the rotation-tracked estimates, verified
residuals and counters; plus acceptance criteria 6 / 8 (acceptance.cpp:
243-330): the baseline converges on none of the 50 grid-family systems and
spends at least 10x the recycled solver's inner products."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def _csr(sk, M):
    off, col, val = M.csr()
    return sk.SparseMatrix(M.rows, M.cols, off, col, val)


def _dense(sk, O, A):
    S = sp.csr_matrix(A)
    return (sk.SparseMatrix(A.shape[0], A.shape[1], S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data),
            O.SparseMatrix.from_dense(A))


def _compare(rep, ref, rtol=1e-6):
    assert rep.status == ref.status
    assert rep.iterations == ref.iterations and rep.cycles == ref.cycles
    assert rep.counters == ref.counters
    assert rep.notes == ref.notes
    assert rep.rhs_norm == pytest.approx(ref.rhs_norm, rel=1e-12)
    got = np.array([v for _, v in rep.sketched_residuals])
    want = np.array([v for _, v in ref.sketched_residuals])
    assert [i for i, _ in rep.sketched_residuals] == [i for i, _ in ref.sketched_residuals]
    np.testing.assert_allclose(got, want, rtol=rtol, atol=1e-13 * ref.rhs_norm)
    for (i1, r1), (i2, r2) in zip(rep.true_residuals, ref.true_residuals):
        assert i1 == i2 and r1 == pytest.approx(r2, rel=rtol, abs=1e-13 * ref.rhs_norm)


@pytest.mark.parametrize("m,restarts", [(40, 30), (7, 200), (100, 5)])
def test_baseline_matches_oracle(sk, O, m, restarts):
    M = O.gen_convdiff(30, -10.0)
    A = _csr(sk, M)
    b = O.gaussian_vector(900, 5)
    xo, ro = O.baseline_gmres(M, b, m=m, tol=1e-8, max_restarts=restarts)
    res = sk.baseline_gmres(A, b, sk.BaselineConfig(m=m, tol=1e-8, max_restarts=restarts))
    _compare(res.report, ro)
    np.testing.assert_allclose(res.x, xo, rtol=1e-6, atol=1e-9 * np.linalg.norm(xo))


def test_baseline_x0_and_device_buffers(sk, O):
    import torch
    M = O.gen_convdiff(25, 15.0)
    A = _csr(sk, M)
    b = O.gaussian_vector(625, 11)
    x0 = 0.1 * O.gaussian_vector(625, 12)
    xo, ro = O.baseline_gmres(M, b, m=30, tol=1e-9, max_restarts=50, x0=x0)
    res = sk.baseline_gmres(A, torch.from_numpy(b).cuda(), sk.BaselineConfig(m=30, tol=1e-9, max_restarts=50),
                            x0=torch.from_numpy(x0).cuda())
    _compare(res.report, ro)
    assert res.report.counters["matvecs"] == ro.counters["matvecs"]  # includes the A x0 product
    np.testing.assert_allclose(res.x.cpu().numpy(), xo, rtol=1e-6, atol=1e-9 * np.linalg.norm(xo))


def test_baseline_edge_cases(sk, O):
    n = 30
    A3, O3 = _dense(sk, O, 3.0 * np.eye(n))
    b = O.gaussian_vector(n, 9)
    res = sk.baseline_gmres(A3, b, sk.BaselineConfig(m=5, tol=1e-10))
    assert res.report.status == "converged" and res.report.iterations == 1
    np.testing.assert_allclose(res.x, b / 3.0, rtol=1e-14)
    res = sk.baseline_gmres(A3, np.zeros(n), sk.BaselineConfig(m=5, tol=1e-10))
    assert res.report.status == "converged" and res.report.iterations == 0 and res.report.cycles == 0
    # cyclic shift: no progress before step n -> diverged, same note as the reference
    P = np.roll(np.eye(n), 1, axis=0)
    e0 = np.zeros(n)
    e0[0] = 1.0
    AP, OP = _dense(sk, O, P)
    res = sk.baseline_gmres(AP, e0, sk.BaselineConfig(m=10, tol=1e-8, max_restarts=5))
    _, ro = O.baseline_gmres(OP, e0, m=10, tol=1e-8, max_restarts=5)
    _compare(res.report, ro)
    assert res.report.status == "diverged"
    # n-step shift with m = n: the Krylov space is invariant at step n
    res = sk.baseline_gmres(AP, e0, sk.BaselineConfig(m=n, tol=1e-8, max_restarts=2))
    _, ro = O.baseline_gmres(OP, e0, m=n, tol=1e-8, max_restarts=2)
    _compare(res.report, ro)
    with pytest.raises(ValueError):
        sk.baseline_gmres(A3, b, sk.BaselineConfig(m=0))
    with pytest.raises(ValueError):
        sk.baseline_gmres(A3, b, sk.BaselineConfig(m=256))  # device limit
    res = sk.baseline_gmres(A3, b, sk.BaselineConfig(m=255, tol=1e-10))
    assert res.report.status == "converged"


def test_baseline_long_cycle_m255(sk, O):
    M = O.gen_convdiff(40, -30.0)
    A = _csr(sk, M)
    b = O.gaussian_vector(1600, 21)
    xo, ro = O.baseline_gmres(M, b, m=255, tol=1e-10, max_restarts=3)
    res = sk.baseline_gmres(A, b, sk.BaselineConfig(m=255, tol=1e-10, max_restarts=3))
    _compare(res.report, ro, rtol=1e-5)


def test_acceptance_baseline_stalls_and_inner_product_gap(sk, O):
    """Criteria 6 (baseline part) and 8 on the grid family (acceptance.cpp:267-283, 321-330)."""
    A = _csr(sk, O.gen_neumann(103, 1e-4))
    n = A.rows
    rhs = [sk.gaussian_vector(n, 2026 + i) for i in range(50)]
    cfg = sk.SolverConfig(m=100, t=2, k=20, s=1200, tol=1e-6, max_restarts=10)
    out = sk.solve_sequence([sk.ProblemInstance(A, b, target_tol=1e-6) for b in rhs], cfg, shared_matrix=True)
    recycled_ips = sum(r.counters["inner_products"] for r in out.reports)
    bcfg = sk.BaselineConfig(m=100, tol=1e-6, max_restarts=10)
    base = [sk.baseline_gmres(A, b, bcfg).report for b in rhs]
    assert sum(r.status == "converged" for r in base) == 0
    baseline_ips = sum(r.counters["inner_products"] for r in base)
    assert baseline_ips / recycled_ips >= 10.0
    # the device baseline follows the oracle on the first system
    Mo = O.gen_neumann(103, 1e-4)
    _, ro = O.baseline_gmres(Mo, rhs[0], m=100, tol=1e-6, max_restarts=10)
    _compare(base[0], ro, rtol=1e-5)
