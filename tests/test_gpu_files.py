"""Files on the device path: a Matrix Market operator
solves exactly like the same CSR uploaded directly, and a recycle space
saved to SKRYRCY1 and loaded back (recycle.hpp:337-390) drives the next solve
identically to the in-memory space (the reference's --save-space /
--load-space flow, test_campaign.cpp:180-200)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_matrix_market_operator_solves_like_direct_csr(sk, tmp_path):
    off, col, val = sk.gen_convdiff(40, -20.0)
    n = 1600
    path = str(tmp_path / "A.mtx")
    sk.write_matrix_market(path, n, n, off, col, val)
    A1 = sk.SparseMatrix(n, n, off, col, val)
    A2 = sk.SparseMatrix.from_matrix_market(path)
    assert (A2.rows, A2.cols, A2.nnz) == (n, n, len(val))
    x = sk.gaussian_vector(n, 5)
    assert np.array_equal(A1.apply(x), A2.apply(x))
    b = sk.gaussian_vector(n, 6)
    cfg = sk.SolverConfig(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=20)
    r1, r2 = sk.solve(A1, b, cfg), sk.solve(A2, b, cfg)
    assert r1.report.iterations == r2.report.iterations and np.array_equal(r1.x, r2.x)


def test_recycle_space_save_load_round_trip(sk, tmp_path):
    off, col, val = sk.gen_convdiff(40, -20.0)
    n = 1600
    A = sk.SparseMatrix(n, n, off, col, val)
    cfg = sk.SolverConfig(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=20)
    space = sk.RecycleSpace()
    sk.solve(A, sk.gaussian_vector(n, 1), cfg, space=space)
    assert space.dim() > 0
    path = str(tmp_path / "space.bin")
    sk.save_recycle_space(path, space)
    f = sk.read_space_file(path)
    U, SU, SAU = space.U, space.SU, space.SAU
    assert f["k"] == space.dim() and f["n"] == n and f["s"] == 80
    assert np.array_equal(f["U"], U) and np.array_equal(f["SU"], SU) and np.array_equal(f["SAU"], SAU)
    loaded = sk.load_recycle_space(path)
    assert loaded.dim() == space.dim() and loaded.provenance == space.provenance
    b2 = sk.gaussian_vector(n, 2)
    r_mem = sk.solve(A, b2, cfg, space=space)
    r_file = sk.solve(A, b2, cfg, space=loaded)
    assert r_mem.report.iterations == r_file.report.iterations
    np.testing.assert_allclose(r_file.x, r_mem.x, rtol=1e-12, atol=1e-14 * np.linalg.norm(r_mem.x))
