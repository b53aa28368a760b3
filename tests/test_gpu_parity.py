"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Tolerances follow BASELINE.json's north_star: per-kernel SpMV / sketch
outputs within 1e-12 relative (fp64), sketch rows/signs bit-identical,
solver status equal with iteration counts within ±2%.
"""
import numpy as np
import scipy.sparse as sp
import pytest

pytestmark = pytest.mark.gpu

REL = 1e-12


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def random_matrix(O, n, seed):
    """test_solver.cpp:27-34: gaussian + n I, column-major draw order."""
    g = O.gaussian_vector(n * n, seed)
    A = g.reshape(n, n).T.copy()
    A[np.diag_indices(n)] += n
    return A


def to_both(sk, O, off, col, val, rows, cols):
    return sk.SparseMatrix(rows, cols, off, col, val), O.SparseMatrix.from_csr(rows, cols, off, col, val)


# ----------------------------------------------------------------------- SpMV

@pytest.mark.parametrize("case", ["c1", "conv3d", "random", "dense", "empty_rows"])
def test_spmv_matches_oracle(sk, O, case):
    rng = np.random.default_rng(7)
    if case == "c1":
        off, col, val = O.gen_convdiff(100, -50.0).csr()
        off, col, val, n = off, col, -val, 10000
    elif case == "conv3d":
        off, col, val = O.gen_convdiff3d(40, 100.0, 50.0, 25.0).csr()
        n = 40 ** 3
    elif case == "random":
        n = 5000
        lens = rng.integers(0, 40, n)
        rows = np.repeat(np.arange(n), lens)
        cols_ = rng.integers(0, n, rows.size)
        M = O.SparseMatrix.from_triplets(n, n, rows, cols_, rng.standard_normal(rows.size))
        off, col, val = M.csr()
    elif case == "dense":
        n = 70
        off, col, val = O.SparseMatrix.from_dense(random_matrix(O, n, 3)).csr()
    else:
        n = 300
        rows = rng.integers(0, n, 600)
        rows = rows[rows % 3 != 0]
        M = O.SparseMatrix.from_triplets(n, n, rows, rng.integers(0, n, rows.size), rng.standard_normal(rows.size))
        off, col, val = M.csr()
    A, Ao = to_both(sk, O, off, col, val, n, n)
    for seed in (1, 2):
        x = O.gaussian_vector(n, seed)
        assert rel(A.apply(x), Ao.apply(x)) <= REL


@pytest.mark.parametrize("offsets,rows,cols,fmt", [
    ((-1, 0, 1), 1000, 1000, "dia"),                      # runtime D = 3
    ((-200, -1, 0, 1, 200), 4000, 4000, "dia"),           # compile-time D = 5
    (tuple(range(-4, 5)), 2000, 2000, "dia"),             # runtime D = 9
    (tuple(range(-8, 9)), 2000, 2000, "sell"),            # 17 diagonals: SELL-32
    ((-3, 0, 2, 7), 300, 500, "dia"),                     # rectangular
])
def test_banded_storage_forms_match_oracle(sk, O, offsets, rows, cols, fmt):
    """SELL-DIA (compile-time and runtime diagonal counts, rectangular, gaps at
    the matrix edges) and the SELL-32 fallback against the oracle's CSR."""
    rng = np.random.default_rng(len(offsets) + rows)
    r, c = [], []
    for o in offsets:
        i = np.arange(max(0, -o), min(rows, cols - o))
        r.append(i)
        c.append(i + o)
    r, c = np.concatenate(r), np.concatenate(c)
    M = O.SparseMatrix.from_triplets(rows, cols, r, c, rng.standard_normal(r.size))
    off, col, val = M.csr()
    A = sk.SparseMatrix(rows, cols, off, col, val)
    assert A.storage["format"] == fmt
    x = O.gaussian_vector(cols, 9)
    assert rel(A.apply(x), M.apply(x)) <= REL


def test_device_generated_operator_matches_host_csr(sk, O):
    n = 48
    Ad = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0)
    off, col, val = sk.gen_convdiff3d(n, 100.0, 50.0, 25.0)
    Ah = sk.SparseMatrix(n ** 3, n ** 3, off, col, val)
    assert Ad.nnz == Ah.nnz == len(val)
    x = O.gaussian_vector(n ** 3, 5)
    yd, yh = Ad.apply(x), Ah.apply(x)
    assert np.array_equal(yd, yh)


def test_spmv_rejects_bad_input(sk):
    with pytest.raises(ValueError, match="offsets must start at 0"):
        sk.SparseMatrix(2, 2, [1, 1, 2], [0], [1.0])
    with pytest.raises(ValueError, match="not strictly increasing in row 0"):
        sk.SparseMatrix(2, 2, [0, 2, 2], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError, match="non-finite value in row 1"):
        sk.SparseMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, np.inf])
    A = sk.SparseMatrix(2, 3, [0, 1, 2], [0, 2], [1.0, 2.0])
    with pytest.raises(ValueError, match="3 columns but vector has 2 entries"):
        A.apply(np.ones(2))


# --------------------------------------------------------------------- sketches

@pytest.mark.parametrize("n,s,seed", [(200, 48, 31), (4096, 240, 0x5EED), (2 ** 21, 240, 0x5EED), (10000, 120, 0)])
def test_srdct_rows_and_signs_bit_exact(sk, O, n, s, seed):
    S = sk.SketchOperator.subsampled_dct(n, s, seed)
    So = O.SketchOperator.subsampled_dct(n, s, seed)
    assert np.array_equal(S.rows(), So.rows())
    assert np.array_equal(S.signs(), So.signs())


@pytest.mark.parametrize("n,s", [(200, 48), (256, 64), (1000, 120), (10000, 120), (65536, 240), (2 ** 20, 140),
                                 (2 ** 21, 240), (3 * 2 ** 15, 200), (997, 60), (10609, 1200), (12345, 777),
                                 (2 ** 13 + 1, 300)])
def test_srdct_apply_matches_oracle(sk, O, n, s):
    S = sk.SketchOperator.subsampled_dct(n, s, 0x5EED)
    So = O.SketchOperator.subsampled_dct(n, s, 0x5EED)
    for seed in (11, 12):
        x = O.gaussian_vector(n, seed)
        assert rel(S.apply(x), So.apply(x)) <= REL


def test_srdct_matches_scipy_dct(sk, O):
    import scipy.fft
    n, s = 4096, 100
    S = sk.SketchOperator.subsampled_dct(n, s, 99)
    x = O.gaussian_vector(n, 3)
    ref = np.sqrt(n / s) * scipy.fft.dct(S.signs() * x, type=2, norm="ortho")[S.rows()]
    assert rel(S.apply(x), ref) <= REL


@pytest.mark.parametrize("n,s,zeta", [(10000, 120, 8), (4097, 240, 8), (1000, 37, 5), (64, 16, 16)])
def test_sparse_sign_matches_oracle(sk, O, n, s, zeta):
    S = sk.SketchOperator.sparse_sign(n, s, 0x5EED, zeta)
    So = O.SketchOperator.sparse_sign(n, s, 0x5EED, zeta)
    x = O.gaussian_vector(n, 4)
    assert rel(S.apply(x), So.apply(x)) <= REL


def test_identity_sketch_passes_through(sk, O):
    S = sk.SketchOperator.identity(40)
    x = O.gaussian_vector(40, 8)
    assert np.array_equal(S.apply(x), x)


def test_sketch_is_linear_and_deterministic(sk, O):
    n = 2 ** 16
    S = sk.SketchOperator.subsampled_dct(n, 240, 7)
    a, b = O.gaussian_vector(n, 1), O.gaussian_vector(n, 2)
    sa, sb, sab = S.apply(a), S.apply(b), S.apply(2.0 * a - 3.0 * b)
    assert np.linalg.norm(sab - (2.0 * sa - 3.0 * sb)) <= 1e-13 * np.linalg.norm(sab)
    assert np.array_equal(S.apply(a), sa)


# --------------------------------------------------------------- Arnoldi steps

def krylov(sk, A, S, r0, t, m, steps=None, btol=1e-14):
    import ctypes as C
    n, s = A.local_rows, S.sketch_dim
    V = np.zeros((m + 1) * n)
    H = np.zeros((m + 1) * m)
    SV = np.zeros(s * (m + 1))
    SAV = np.zeros(s * m)
    j, br, rn = C.c_int64(), C.c_int(), C.c_double()
    cnt = np.zeros(3, dtype=np.int64)
    r0 = np.ascontiguousarray(r0, dtype=np.float64)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    sk._check(sk._lib.sdr_krylov_run(A.ctx._h, A._h, S._h, p(r0), t, m, m if steps is None else steps, btol, p(V),
                                     p(H), p(SV), p(SAV), C.byref(j), C.byref(br), C.byref(rn), p(cnt)))
    return dict(V=V.reshape(m + 1, n).T, H=H.reshape(m, m + 1).T, SV=SV.reshape(m + 1, s).T,
                SAV=SAV.reshape(m, s).T, j=j.value, breakdown=bool(br.value), r0_norm=rn.value,
                counters=tuple(int(c) for c in cnt))


@pytest.mark.parametrize("t", [1, 2, 3])
def test_arnoldi_matches_oracle(sk, O, t):
    n, m, s = 60, 12, 40
    M = random_matrix(O, n, 17)
    A, Ao = sk.SparseMatrix.from_dense(M), O.SparseMatrix.from_dense(M)
    S, So = sk.SketchOperator.subsampled_dct(n, s, 23), O.SketchOperator.subsampled_dct(n, s, 23)
    r0 = O.gaussian_vector(n, 29)
    g = krylov(sk, A, S, r0, t, m)
    o = O.run_arnoldi(Ao, r0, So, t, m)
    assert g["j"] == o.j == m and not g["breakdown"]
    assert g["counters"] == tuple(o.counters)
    assert rel(g["H"], o.H) <= 1e-12
    assert rel(g["SV"], o.SV) <= 1e-12
    assert rel(g["SAV"], o.SAV) <= 1e-11
    assert rel(g["V"], o.V) <= 1e-12
    # recurrence A v_q = V H(:, q) and band structure (test_arnoldi.cpp:34-52)
    for q in range(m):
        lhs = M @ g["V"][:, q]
        assert np.linalg.norm(lhs - g["V"][:, : q + 2] @ g["H"][: q + 2, q]) <= 1e-12 * np.linalg.norm(lhs)
        assert np.all(g["H"][: max(0, q - t + 1), q] == 0.0)


def test_arnoldi_c1_operator_long_window(sk, O):
    off, col, val = O.gen_convdiff(100, -50.0).csr()
    A, Ao = to_both(sk, O, off, col, -val, 10000, 10000)
    S, So = sk.SketchOperator.subsampled_dct(10000, 120, 0x5EED), O.SketchOperator.subsampled_dct(10000, 120, 0x5EED)
    r0 = O.gaussian_vector(10000, 0)
    g = krylov(sk, A, S, r0, 2, 50)
    o = O.run_arnoldi(Ao, r0, So, 2, 50)
    assert rel(g["H"], o.H) <= 1e-10
    assert rel(g["SV"], o.SV) <= 1e-10


def test_arnoldi_breakdown_on_invariant_subspace(sk, O):
    n = 20
    A = sk.SparseMatrix.from_dense(2.5 * np.eye(n))
    S = sk.SketchOperator.subsampled_dct(n, 10, 3)
    g = krylov(sk, A, S, O.gaussian_vector(n, 31), 2, 5)
    assert g["breakdown"] and g["j"] == 1
    assert g["H"][1, 0] == 0.0
    assert abs(g["H"][0, 0] - 2.5) <= 1e-12 * 2.5


def test_arnoldi_full_window_is_dense_arnoldi(sk, O):
    n, m = 30, 8
    M = random_matrix(O, n, 11)
    A = sk.SparseMatrix.from_dense(M)
    S = sk.SketchOperator.identity(n)
    r0 = O.gaussian_vector(n, 13)
    g = krylov(sk, A, S, r0, m, m)
    V = g["V"][:, : m + 1]
    assert np.linalg.norm(V.T @ V - np.eye(m + 1)) < 1e-8


def test_zero_start_is_domain_error(sk):
    A = sk.SparseMatrix.from_dense(np.eye(8))
    S = sk.SketchOperator.identity(8)
    with pytest.raises(ArithmeticError):
        krylov(sk, A, S, np.zeros(8), 1, 4)


@pytest.mark.parametrize("kind", ["dia7", "dia5", "sell", "csr_wide"])
@pytest.mark.parametrize("nb", [1, 5, 8, 13, 20])
def test_spmm_columns_equal_spmv_bitwise(sk, O, kind, nb):
    """The batched refresh product (recycle.hpp:309-316) per column equals the single SpMV exactly."""
    if kind == "dia7":
        off, col, val = sk.gen_convdiff3d(12, 100.0, 50.0, 25.0)
        n = 12 ** 3
    elif kind == "dia5":
        off, col, val = sk.gen_convdiff(30, -20.0)
        n = 900
    else:
        rng = np.random.default_rng(3)
        n = 700
        per = 9 if kind == "sell" else 40
        r = np.repeat(np.arange(n), per)
        c = rng.integers(0, n, n * per)
        M = O.SparseMatrix.from_triplets(n, n, r, c, rng.standard_normal(n * per))
        off, col, val = M.csr()
    A = sk.SparseMatrix(n, n, off, col, val)
    X = np.asfortranarray(np.stack([O.gaussian_vector(n, 100 + q) for q in range(nb)], axis=1))
    Y = A.apply_batch(X)
    for q in range(nb):
        assert np.array_equal(Y[:, q], A.apply(X[:, q]))


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("n,k1,k2,nout", [(1000, 7, 3, 5), (4096, 100, 20, 20), (8191, 50, 0, 21), (300, 33, 31, 24),
                                          (257, 1, 0, 1), (65536, 121, 20, 12)])
def test_recycle_product_kernels(sk, kernel, n, k1, k2, nout):
    """U_new = [V U] C with fused column norms (recycle.hpp:257-280 product)."""
    import ctypes as C
    if kernel == 0 and (n % 2 or nout > 24):
        pytest.skip("k_tsgemm needs an even row count")
    rng = np.random.default_rng(n + k1)
    lda1, lda2 = n + (n % 2) + 32, n + (n % 2) + 64
    A1 = rng.standard_normal((k1, lda1)).T.copy(order="F")
    A2 = rng.standard_normal((max(k2, 1), lda2)).T.copy(order="F")
    B = np.asfortranarray(rng.standard_normal((k1 + k2, nout)))
    Cm = np.zeros((n, nout), order="F")
    nr = np.zeros(nout)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    sk._check(sk._lib.sdr_debug_block_product(sk.default_context()._h, kernel, n, p(A1), lda1, k1, p(A2), lda2, k2,
                                              p(B), nout, p(Cm), n, p(nr)))
    ref = A1[:n, :k1] @ B[:k1] + (A2[:n, :k2] @ B[k1:] if k2 else 0.0)
    assert np.linalg.norm(Cm - ref) <= 1e-13 * np.linalg.norm(ref)
    np.testing.assert_allclose(nr, (ref ** 2).sum(axis=0), rtol=1e-12)


def _complex_realified(rng, nc, per_row, zero_imag_diag=True):
    """Random complex CSR -> its real-equivalent (interleaved (re, im)) CSR."""
    rows, cols, vals = [], [], []
    for p in range(nc):
        qs = np.unique(np.concatenate([[p], rng.integers(0, nc, per_row)]))
        for q in qs:
            a = rng.standard_normal() + (4.0 if q == p else 0.0)
            b = 0.0 if (q == p and zero_imag_diag) else rng.standard_normal()
            for rr, cc, vv in ((2 * p, 2 * q, a), (2 * p, 2 * q + 1, -b), (2 * p + 1, 2 * q, b), (2 * p + 1, 2 * q + 1, a)):
                if vv != 0.0:
                    rows.append(rr)
                    cols.append(cc)
                    vals.append(vv)
    M = sp.csr_matrix((vals, (rows, cols)), shape=(2 * nc, 2 * nc))
    M.sort_indices()
    return M


def test_complex_spmv_zsell_matches_real_path(sk, O):
    """ZSELL (complex-fp64 SpMV on interleaved vectors) equals the real SELL
    path on the realified operator bit for bit, and the complex product."""
    import os
    import subprocess
    import sys
    rng = np.random.default_rng(5)
    nc = 3000
    M = _complex_realified(rng, nc, 8)
    A = sk.SparseMatrix(2 * nc, 2 * nc, M.indptr.astype(np.int64), M.indices.astype(np.int64), M.data)
    assert A.storage["format"] == "zsell"
    x = O.gaussian_vector(2 * nc, 3)
    y = A.apply(x)
    ref = M @ x
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)
    # the same operator with ZSELL off (real SELL-32) in a fresh process: identical bits
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); import paper_2311_14206_b200 as sk; "
            "d = np.load(sys.argv[1]); A = sk.SparseMatrix(d['n'], d['n'], d['o'], d['c'], d['v']); "
            "assert A.storage['format'] == 'sell'; np.save(sys.argv[2], A.apply(d['x']))")
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        np.savez(os.path.join(td, "in.npz"), n=2 * nc, o=M.indptr.astype(np.int64), c=M.indices.astype(np.int64),
                 v=M.data, x=x)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        p = subprocess.run([sys.executable, "-c", code, os.path.join(td, "in.npz"), os.path.join(td, "out.npy")],
                           cwd=root, env=dict(os.environ, SDR_ZSELL="0"), capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        y_real = np.load(os.path.join(td, "out.npy"))
    assert np.array_equal(y, y_real)
    # as a complex product
    z = x[0::2] + 1j * x[1::2]
    Z = (M[0::2, 0::2] + 1j * M[1::2, 0::2])
    yz = Z @ z
    np.testing.assert_allclose(y[0::2] + 1j * y[1::2], yz, rtol=1e-12, atol=1e-12 * np.abs(yz).max())


def test_complex_structure_detection_rejects_real_operators(sk):
    off, col, val = sk.gen_convdiff(30, -20.0)
    A = sk.SparseMatrix(900, 900, off, col, val)
    assert A.storage["format"] != "zsell"
    rng = np.random.default_rng(6)
    M = _complex_realified(rng, 200, 4)
    M = M.tolil()
    M[0, 1] += 1e-3  # breaks one 2x2 block
    M = M.tocsr()
    B = sk.SparseMatrix(400, 400, M.indptr.astype(np.int64), M.indices.astype(np.int64), M.data)
    assert B.storage["format"] == "sell"


def test_complex_system_solves_through_zsell(sk, O):
    """A complex system in real-equivalent form: the solve on ZSELL storage
    equals the oracle's real GMRES-SDR on the realified CSR."""
    rng = np.random.default_rng(8)
    nc = 2000
    M = _complex_realified(rng, nc, 6)
    off, col, val = M.indptr.astype(np.int64), M.indices.astype(np.int64), M.data
    A = sk.SparseMatrix(2 * nc, 2 * nc, off, col, val)
    assert A.storage["format"] == "zsell"
    b = O.gaussian_vector(2 * nc, 9)
    cfg = sk.SolverConfig(m=40, k=8, t=3, s=100, tol=1e-10, max_restarts=20)
    r = sk.solve(A, b, cfg)
    xo, ro = O.solve(O.SparseMatrix.from_csr(2 * nc, 2 * nc, off, col, val), b,
                     O.SolverConfig(m=40, k=8, t=3, s=100, tol=1e-10, max_restarts=20))
    assert r.report.status == ro.status == "converged"
    assert abs(r.report.iterations - ro.iterations) <= max(1, 0.02 * ro.iterations)
    assert np.linalg.norm(b - M @ r.x) <= 1e-10 * np.linalg.norm(b) * (1 + 1e-9)


@pytest.mark.parametrize("rows,cols,density", [(1, 1, 1.0), (5, 5, 0.3), (31, 31, 0.2), (33, 7, 0.5), (7, 33, 0.5),
                                               (64, 64, 0.0), (97, 97, 0.05)])
def test_spmv_small_and_degenerate_shapes(sk, O, rows, cols, density):
    """Partial slices (rows not a multiple of 32), a single row, rectangular
    blocks and an operator with no stored entry at all."""
    rng = np.random.default_rng(rows * 131 + cols)
    mask = rng.random((rows, cols)) < density
    D = np.where(mask, rng.standard_normal((rows, cols)), 0.0)
    S = sp.csr_matrix(D)
    A = sk.SparseMatrix(rows, cols, S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data)
    x = O.gaussian_vector(cols, 3)
    y = A.apply(x)
    ref = D @ x
    assert y.shape == (rows,)
    if np.linalg.norm(ref) == 0:
        assert not np.any(y)
    else:
        assert rel(y, ref) <= REL


def test_complex_csr_api(sk, O):
    """sdr_csr_create_complex: complex CSR in, ZSELL operator on interleaved vectors."""
    rng = np.random.default_rng(12)
    nc = 1500
    Z = sp.random(nc, nc, density=0.004, random_state=3, format="csr", dtype=np.float64)
    Z = (Z + 1j * sp.random(nc, nc, density=0.004, random_state=4, format="csr")).tocsr()
    Z = (Z + sp.identity(nc) * (5.0 + 0.5j)).tocsr()
    Z.sort_indices()
    A = sk.SparseMatrix.from_complex(nc, nc, Z.indptr, Z.indices, Z.data)
    assert A.storage["format"] == "zsell" and A.rows == 2 * nc
    z = rng.standard_normal(nc) + 1j * rng.standard_normal(nc)
    y = A.apply_complex(z)
    ref = Z @ z
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    with pytest.raises(ValueError, match="not strictly increasing"):
        sk.SparseMatrix.from_complex(2, 2, [0, 2, 2], [1, 1], np.array([1 + 1j, 2.0]))
