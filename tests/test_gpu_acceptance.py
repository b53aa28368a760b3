"""End-to-end acceptance gates on the GPU path (proj/tests/acceptance.cpp):
criterion 6 (grid family: every recycled solve converges, the last system
needs fewer steps than the first) and criterion 9 (convection variants:
refreshing the sketched image converges everywhere, carrying a stale image
fails the strongest jump). Operators come from the oracle's restated
generators (test-side inputs only); the solves run through the C-ABI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _csr(sk, M):
    off, col, val = M.csr()
    return sk.SparseMatrix(M.rows, M.cols, off, col, val)


def test_acceptance_grid_family(sk, O):
    """acceptance.cpp:243-288: neumann_sequence(103, 1e-4, 50, 2026, 1e-6),
    m=100 t=2 k=20 s=10(m+k) tol=1e-6 max_restarts=10: 50/50 converge, last < first."""
    A = _csr(sk, O.gen_neumann(103, 1e-4))
    n = A.rows
    probs = [sk.ProblemInstance(A, sk.gaussian_vector(n, 2026 + i), target_tol=1e-6) for i in range(50)]
    cfg = sk.SolverConfig(m=100, t=2, k=20, s=1200, tol=1e-6, max_restarts=10)
    out = sk.solve_sequence(probs, cfg, shared_matrix=True)
    assert all(r.status == "converged" and not r.error for r in out.reports)
    assert out.reports[-1].iterations < out.reports[0].iterations
    for p, x in zip(probs, out.solutions[:5]):
        assert np.linalg.norm(p.rhs - A.apply(x)) <= 1e-6 * np.linalg.norm(p.rhs) * (1 + 1e-9)


def test_acceptance_convection_variants(sk, O):
    """acceptance.cpp:290-320: convdiff_sequence(100, {0, 5, 20}, 1e-2), m=80
    t=2 k=20 s=10(m+k): exact refresh converges 3/3; the inexact (stale image)
    variant does not converge on the last system."""
    mats = [_csr(sk, O.gen_convdiff(100, a)) for a in (0.0, 5.0, 20.0)]
    ones = np.ones(mats[0].rows)
    probs = [sk.ProblemInstance(A, ones, target_tol=1e-2) for A in mats]
    base = dict(m=80, t=2, k=20, s=1000, tol=1e-2, max_restarts=10)
    exact = sk.solve_sequence(probs, sk.SolverConfig(variant="exact", **base))
    assert all(r.status == "converged" and not r.error for r in exact.reports)
    inexact = sk.solve_sequence(probs, sk.SolverConfig(variant="inexact", **base))
    assert len(inexact.reports) == 3 and not inexact.reports[2].error
    assert inexact.reports[2].status != "converged"
