"""Callable operators through the C-ABI (sdr_operator_create_callback):
OperatorRef(rows, cols, Apply) — operator_ref.hpp:22-25, README "Anything
that applies vectors can be an operator".

(a) a callback that wraps the library's own SpMV reproduces the stored-CSR
    solve exactly (same product, same epilogue sums);
(b) a Jacobi-scaled operator D^-1 A (a user preconditioner, applied as a
    torch op on the library's stream) matches the oracle's callable solve
    (status, iterations within ±2 %, counters when equal);
(c) the reference's error behaviour: dimension mismatch, failing callback."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def conv(sk, O, n=16):
    off, col, val = sk.gen_convdiff3d(n, 100.0, 50.0, 25.0)
    N = n ** 3
    return N, off, col, val, sk.SparseMatrix(N, N, off, col, val), O.SparseMatrix.from_csr(N, N, off, col, val)


@pytest.mark.parametrize("sketch", ["srdct", "sparse_sign"])
def test_callable_wrapping_spmv_equals_csr_solve(sk, O, sketch):
    N, off, col, val, A, _ = conv(sk, O)

    def apply(x, y, stream):
        # the library's own product, enqueued on the same (context) stream
        sk._check(sk._lib.sdr_spmv(A.ctx._h, A._h, C.c_void_p(x.ptr), N, C.c_void_p(y.ptr)))

    L = sk.SparseMatrix.from_callable(N, N, apply)
    assert L.storage["format"] == "callable" and L.storage["bytes"] == 0
    S = (sk.SketchOperator.subsampled_dct(N, 80, 0x5EED) if sketch == "srdct"
         else sk.SketchOperator.sparse_sign(N, 80, 0x5EED, 8))
    b = O.gaussian_vector(N, 3)
    cfg = sk.SolverConfig(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=30)
    g = sk.solve(A, b, cfg, sketch=S)
    h = sk.solve(L, b, cfg, sketch=S)
    assert h.report.status == g.report.status == "converged"
    assert h.report.iterations == g.report.iterations
    assert h.report.counters == g.report.counters
    assert np.linalg.norm(h.x - g.x) <= 1e-12 * np.linalg.norm(g.x)


def test_callable_jacobi_scaled_matches_oracle(sk, O):
    torch = pytest.importorskip("torch")
    N, off, col, val, A, Ao = conv(sk, O)
    M = Ao.dense()
    d = np.diag(M).copy()
    dinv = torch.tensor(1.0 / d, dtype=torch.float64, device="cuda")

    def apply(x, y, stream):
        with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
            sk._check(sk._lib.sdr_spmv(A.ctx._h, A._h, C.c_void_p(x.ptr), N, C.c_void_p(y.ptr)))
            y.tensor().mul_(dinv)

    L = sk.SparseMatrix.from_callable(N, N, apply)
    b = O.gaussian_vector(N, 5)
    kw = dict(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=30)
    S, So = sk.SketchOperator.subsampled_dct(N, 80, 0x5EED), O.SketchOperator.subsampled_dct(N, 80, 0x5EED)
    g = sk.solve(L, b, sk.SolverConfig(**kw), sketch=S)

    def apply_host(x, y):
        y[:] = (M @ x) / d

    xo, o = O.solve_callable(N, N, apply_host, b, O.SolverConfig(**kw), sketch=So)
    assert g.report.status == o.status == "converged"
    assert abs(g.report.iterations - o.iterations) <= max(1, 0.02 * o.iterations)
    if g.report.iterations == o.iterations:
        assert g.report.counters == o.counters
    assert np.linalg.norm((M @ g.x) / d - b) <= 1e-8 * np.linalg.norm(b)


def test_callable_errors(sk, O):
    N = 64

    def ok(x, y, stream):
        pass

    L = sk.SparseMatrix.from_callable(N, N, ok)
    with pytest.raises(ValueError, match="OperatorRef::apply: operator has 64 columns but vector has 63 entries"):
        L.apply(np.zeros(63))

    def bad(x, y, stream):
        raise RuntimeError("user failure")

    B = sk.SparseMatrix.from_callable(N, N, bad)
    with pytest.raises(sk.SdrError, match="apply callback"):
        B.apply(np.ones(N))
    R = sk.SparseMatrix.from_callable(N, N + 1, ok)
    with pytest.raises(ValueError, match="square"):
        sk.solve(R, np.ones(N), sk.SolverConfig(m=10, k=2, t=2, s=24, tol=1e-6))


def test_callable_sequence_equals_csr_sequence(sk, O):
    """solve_sequence over callable operators (recycle.hpp:297-318 exact
    refresh applies A to the carried U through the callback, column by
    column) reproduces the stored-CSR sequence: same status, iterations,
    counters and solutions per system."""
    n, count = 12, 4
    N = n ** 3
    mats, calls = [], []
    for i in range(count):
        off, col, val = sk.gen_convdiff3d(n, 100.0 + 10.0 * i, 50.0, 25.0)
        A = sk.SparseMatrix(N, N, off, col, val)
        mats.append(A)

        def apply(x, y, stream, A=A):
            sk._check(sk._lib.sdr_spmv(A.ctx._h, A._h, C.c_void_p(x.ptr), N, C.c_void_p(y.ptr)))

        calls.append(sk.SparseMatrix.from_callable(N, N, apply))
    rhs = [O.gaussian_vector(N, 20 + i) for i in range(count)]
    cfg = sk.SolverConfig(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=30, variant="exact")
    S = sk.SketchOperator.subsampled_dct(N, 80, 0x5EED)
    g = sk.solve_sequence([sk.ProblemInstance(A, b, target_tol=1e-8) for A, b in zip(mats, rhs)], cfg, sketch=S)
    h = sk.solve_sequence([sk.ProblemInstance(L, b, target_tol=1e-8) for L, b in zip(calls, rhs)], cfg, sketch=S)
    assert h.space.dim() == g.space.dim() > 0
    for i, (rg, rh) in enumerate(zip(g.reports, h.reports)):
        assert rh.status == rg.status == "converged", i
        assert rh.iterations == rg.iterations, i
        assert rh.counters == rg.counters, i
        assert np.linalg.norm(h.solutions[i] - g.solutions[i]) <= 1e-12 * np.linalg.norm(g.solutions[i]), i
