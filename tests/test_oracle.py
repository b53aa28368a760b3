"""Pins the CPU oracle (oracle/, the restatement of the reference library)
against the reference's own known-answer tests and properties
(proj/tests/test_rng.cpp, test_sparse.cpp, test_problems.cpp,
test_sketch.cpp, test_arnoldi.cpp, test_recycle.cpp, test_solver.cpp,
test_sequence.cpp, acceptance.cpp). CPU only."""
import numpy as np
import pytest
import scipy.fft
import scipy.linalg as sl


def random_matrix(O, n, seed):
    g = O.gaussian_vector(n * n, seed)
    A = g.reshape(n, n).T.copy()
    A[np.diag_indices(n)] += n
    return A


# --------------------------------------------------------------------- rng

def test_mt19937_64_standard_check_value(O):
    # C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64
    assert int(O.mt_stream(5489, 10000)[-1]) == 9981545732273789042


def test_mt19937_64_seed_5eed(O):
    assert [int(v) for v in O.mt_stream(0x5EED, 2)] == [16228966549159756932, 5963069153190929591]


def test_equal_seeds_identical_streams(O):  # test_rng.cpp:13-22
    assert np.array_equal(O.gaussian_vector(500, 7), O.gaussian_vector(500, 7))
    assert not np.array_equal(O.gaussian_vector(500, 7), O.gaussian_vector(500, 8))


def test_uniform_and_uniform_below(O):  # test_rng.cpp:24-53
    u = O.uniform_stream(3, 20000)
    assert u.min() >= 0.0 and u.max() < 1.0
    v = O.uniform_below_stream(4, 10, 50000).astype(np.int64)
    assert v.min() == 0 and v.max() == 9
    counts = np.bincount(v, minlength=10)
    assert np.all(np.abs(counts - 5000) < 400)
    with pytest.raises(ValueError):
        O.uniform_below_stream(4, 0, 1)


def test_gaussian_moments_and_signs(O):  # test_rng.cpp:55-80
    g = O.gaussian_vector(200000, 11)
    assert abs(g.mean()) < 0.01 and abs(g.var() - 1.0) < 0.01
    s = O.sign_stream(12, 10000)
    assert set(np.unique(s)) == {-1.0, 1.0} and abs(s.mean()) < 0.05


def test_sample_without_replacement(O):  # test_rng.cpp:82-100
    idx = O.sample_without_replacement(1000, 50, 5)
    assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < 1000
    assert np.array_equal(O.sample_without_replacement(7, 7, 1), np.arange(7))
    with pytest.raises(ValueError):
        O.sample_without_replacement(3, 4, 1)


# ------------------------------------------------------------------ sparse

def test_triplet_assembly_sums_duplicates_and_drops_zeros(O):  # test_sparse.cpp:19-32
    A = O.SparseMatrix.from_triplets(3, 3, [0, 0, 1, 2, 2], [0, 0, 1, 2, 2], [1.0, 2.0, 5.0, 1.0, -1.0])
    off, col, val = A.csr()
    assert off.tolist() == [0, 1, 2, 2] and col.tolist() == [0, 1] and val.tolist() == [3.0, 5.0]


def test_apply_matches_dense(O):  # test_sparse.cpp:34-46
    M = random_matrix(O, 30, 3)
    M[M < 0.3] = 0.0
    A = O.SparseMatrix.from_dense(M)
    x = O.gaussian_vector(30, 4)
    assert np.linalg.norm(A.apply(x) - M @ x) <= 1e-14 * np.linalg.norm(M @ x)


def test_malformed_csr_rejected(O):  # test_sparse.cpp:48-84
    with pytest.raises(ValueError, match="offsets must start at 0"):
        O.SparseMatrix.from_csr(2, 2, [1, 1, 2], [0], [1.0])
    with pytest.raises(ValueError, match="not strictly increasing"):
        O.SparseMatrix.from_csr(2, 2, [0, 2, 2], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError, match="out of range"):
        O.SparseMatrix.from_csr(2, 2, [0, 1, 1], [2], [1.0])
    with pytest.raises(ValueError, match="non-finite"):
        O.SparseMatrix.from_csr(2, 2, [0, 1, 1], [0], [np.nan])
    A = O.SparseMatrix.from_csr(2, 3, [0, 1, 2], [0, 2], [1.0, 2.0])
    with pytest.raises(ValueError, match="3 columns but vector has 2 entries"):
        A.apply(np.ones(2))


# ---------------------------------------------------------------- problems

def test_convdiff_coefficients_exact(O):  # test_problems.cpp:41-61
    n, alpha = 4, 3.0
    D = O.gen_convdiff(n, alpha).dense()
    h2, cv = (n + 1) ** 2, alpha * (n + 1) / 2.0
    p = 1 * n + 1
    assert D[p, p] == -4.0 * h2
    assert D[p, p - n] == h2 - cv and D[p, p + n] == h2 + cv
    assert D[p, p - 1] == h2 - cv and D[p, p + 1] == h2 + cv


def test_c1_operator_is_negated_convdiff(O):
    """BASELINE C1: A = -gen_convdiff(100, -50): diag 40804, p±1/p±n = -10201 ∓ 2525."""
    D = O.gen_convdiff(100, -50.0)
    off, col, val = D.csr()
    E = O.gen_convdiff2d(100, 50.0, 50.0)
    off2, col2, val2 = E.csr()
    assert np.array_equal(off, off2) and np.array_equal(col, col2) and np.array_equal(-val, val2)
    row = val2[off2[150]:off2[151]]
    assert sorted(row.tolist()) == sorted([-10201 - 2525.0, -10201 - 2525.0, 40804.0, -10201 + 2525.0,
                                           -10201 + 2525.0])


def test_neumann_rows_sum_to_shift(O):  # test_problems.cpp:16-39
    D = O.gen_neumann(6, 0.25).dense()
    assert np.allclose(D @ np.ones(36), 0.25)


# ------------------------------------------------------------------ sketch

def test_dct_orthonormal_and_fft_equals_direct(O):  # test_sketch.cpp:18-43
    n, s = 200, 48
    f = O.SketchOperator.subsampled_dct(n, s, 31, "fft")
    d = O.SketchOperator.subsampled_dct(n, s, 31, "direct")
    for trial in range(5):
        x = O.gaussian_vector(n, 100 + trial)
        a, b = f.apply(x), d.apply(x)
        assert np.linalg.norm(a - b) <= 1e-12 * (1 + np.linalg.norm(a))
    n = 256
    f = O.SketchOperator.subsampled_dct(n, s, 31, "fft")
    x = O.gaussian_vector(n, 5)
    ref = np.sqrt(n / s) * scipy.fft.dct(f.signs() * x, type=2, norm="ortho")[f.rows()]
    assert np.linalg.norm(f.apply(x) - ref) <= 1e-13 * np.linalg.norm(ref)


def test_dense_realisation_row_gram(O):  # test_sketch.cpp:45-58
    n, s = 96, 24
    S = O.SketchOperator.subsampled_dct(n, s, 5)
    D = S.dense()
    x = O.gaussian_vector(n, 12)
    assert np.linalg.norm(D @ x - S.apply(x)) <= 1e-12 * (1 + np.linalg.norm(x))
    assert np.linalg.norm(D @ D.T - (n / s) * np.eye(s)) < 1e-12 * (n / s)


def test_seed_determines_operator(O):  # test_sketch.cpp:60-69
    x = O.gaussian_vector(128, 55)
    a, b, c = (O.SketchOperator.subsampled_dct(128, 32, sd).apply(x) for sd in (9, 9, 10))
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_unbiased_norms_across_seeds(O):  # test_sketch.cpp:71-82, acceptance.cpp:334-358
    x = O.gaussian_vector(256, 2)
    r = np.mean([np.sum(O.SketchOperator.subsampled_dct(256, 64, 1000 + i).apply(x) ** 2) for i in range(64)])
    assert abs(r / np.sum(x ** 2) - 1.0) < 0.1


def test_invalid_sketch_shapes(O):  # test_sketch.cpp:106-112
    for n, s in ((100, 100), (100, 0)):
        with pytest.raises(ValueError):
            O.SketchOperator.subsampled_dct(n, s, 1)
    with pytest.raises(ValueError):
        O.SketchOperator.identity(0)


def test_sparse_sign_properties(O):
    """New map: ζ distinct rows per column, one per block,
    values ±1/√ζ, E||Sx||^2 = ||x||^2, linear, seed-determined."""
    n, s, z = 2000, 120, 8
    S = O.SketchOperator.sparse_sign(n, s, 7, z)
    rows, signs = S.sparse_entries(0, n, z)
    for l in range(z):
        lo, hi = (l * s) // z, ((l + 1) * s) // z
        assert np.all((rows[:, l] >= lo) & (rows[:, l] < hi))
    assert set(np.unique(signs)) == {-1.0, 1.0}
    D = S.dense()
    assert np.allclose(np.sum(D != 0, axis=0), z) and np.allclose(np.abs(D[D != 0]), 1 / np.sqrt(z))
    x, y = O.gaussian_vector(n, 1), O.gaussian_vector(n, 2)
    assert np.linalg.norm(S.apply(2 * x - y) - (2 * S.apply(x) - S.apply(y))) <= 1e-13 * np.linalg.norm(S.apply(x))
    r = np.mean([np.sum(O.SketchOperator.sparse_sign(n, s, 100 + i, z).apply(x) ** 2) for i in range(40)])
    assert abs(r / np.sum(x ** 2) - 1.0) < 0.1
    # rows within a block and signs are uniform (15-bit fields: bias <= 15/32768)
    big = O.SketchOperator.sparse_sign(60000, s, 11, z)
    rows, signs = big.sparse_entries(0, 60000, z)
    counts = np.bincount((rows[:, 3] - (3 * s) // z).ravel(), minlength=s // z)
    assert counts.min() > 0.9 * counts.mean() and counts.max() < 1.1 * counts.mean()
    assert abs(np.mean(signs)) < 0.02


# ----------------------------------------------------------------- arnoldi

def test_truncated_recurrence_and_band(O):  # test_arnoldi.cpp:34-52
    n, m, t = 40, 10, 2
    M = random_matrix(O, n, 3)
    st = O.run_arnoldi(O.SparseMatrix.from_dense(M), O.gaussian_vector(n, 7), O.SketchOperator.subsampled_dct(n, 30, 5),
                       t, m)
    assert st.j == m and not st.breakdown
    for q in range(m):
        lhs = M @ st.V[:, q]
        assert np.linalg.norm(lhs - st.V[:, : q + 2] @ st.H[: q + 2, q]) <= 1e-12 * np.linalg.norm(lhs)
        assert np.all(st.H[: max(0, q - t + 1), q] == 0.0)


def test_sketched_blocks_and_exact_counters(O):  # test_arnoldi.cpp:70-95
    n, m, t = 60, 12, 3
    M = random_matrix(O, n, 17)
    S = O.SketchOperator.subsampled_dct(n, 40, 23)
    st = O.run_arnoldi(O.SparseMatrix.from_dense(M), O.gaussian_vector(n, 29), S, t, m)
    for q in range(m + 1):
        sv = S.apply(st.V[:, q])
        assert np.linalg.norm(st.SV[:, q] - sv) <= 1e-13 * (1 + np.linalg.norm(sv))
    for q in range(m):
        sav = S.apply(M @ st.V[:, q])
        assert np.linalg.norm(st.SAV[:, q] - sav) <= 1e-11 * (1 + np.linalg.norm(sav))
    assert st.counters[2] == m + 1 and st.counters[0] == m
    assert st.counters[1] == 1 + sum(min(t, q + 1) + 2 for q in range(m))


def test_breakdown_on_invariant_subspace(O):  # test_arnoldi.cpp:97-115
    n = 20
    st = O.run_arnoldi(O.SparseMatrix.from_dense(2.5 * np.eye(n)), O.gaussian_vector(n, 31),
                       O.SketchOperator.subsampled_dct(n, 10, 3), 2, 5)
    assert st.breakdown and st.j == 1 and st.H[1, 0] == 0.0
    assert st.H[0, 0] == pytest.approx(2.5, rel=1e-12)


# ----------------------------------------------------------------- recycle

def test_harmonic_conjugate_pair_extends(O):  # test_recycle.cpp:131-167
    rng = np.random.default_rng(55)
    Q = np.linalg.qr(rng.standard_normal((4, 4)))[0]
    T0 = np.array([[3.0, 0, 0, 0], [0, 2.0, 1.0, 0], [0, -1.0, 2.0, 0], [0, 0, 0, 0.5]])
    # build SAW = U diag(1) V^T and SW with u^T SW v = Q T0 Q^T
    U = np.linalg.qr(rng.standard_normal((20, 4)))[0]
    Vv = np.linalg.qr(rng.standard_normal((10, 4)))[0]
    SAW = U @ Vv.T
    SW = U @ (Q @ T0 @ Q.T) @ Vv.T
    h = O.harmonic(SAW, SW, 2)
    assert h["k_effective"] == 3 and h["pair_extended"] and not h["rank_limited"]
    assert abs(np.sum(h["mu"]) - 7.0) <= 1e-10 and abs(np.prod(h["mu"]) - 15.0) <= 1e-9


def test_rank_deficient_pencil_shrinks(O):  # test_recycle.cpp:169-185
    rng = np.random.default_rng(58)
    SAW = np.linalg.qr(rng.standard_normal((15, 2)))[0] @ np.linalg.qr(rng.standard_normal((6, 2)))[0].T
    h = O.harmonic(SAW, rng.standard_normal((15, 6)), 5)
    assert h["rank"] == 2 and h["rank_limited"] and h["k_effective"] <= 2


# ------------------------------------------------------------------ solver

def test_identity_sketch_equals_dense_gmres(O):  # test_solver.cpp:38-81, acceptance criterion 1
    n, m = 40, 20
    M = random_matrix(O, n, 81)
    b = O.gaussian_vector(n, 82)
    cfg = O.SolverConfig(m=m, t=m, k=0, s=2 * m, tol=1e-8, safety_init=1.0, max_restarts=2)
    x, rep = O.solve(O.SparseMatrix.from_dense(M), b, cfg, sketch=O.SketchOperator.identity(n))
    assert rep.status == "converged" and rep.cycles == 1
    # dense GMRES residuals from an explicit Krylov basis (numpy)
    K = np.empty((n, rep.iterations))
    v = b / np.linalg.norm(b)
    for j in range(rep.iterations):
        K[:, j] = v
        v = M @ v
        v = v / np.linalg.norm(v)
    for (it, val) in rep.sketched_residuals:
        Q = sl.orth(K[:, :it])
        y = np.linalg.lstsq(M @ Q, b, rcond=None)[0]
        assert abs(val - np.linalg.norm(b - M @ Q @ y)) <= 1e-8 * np.linalg.norm(b)
    assert rep.final_relative_residual == pytest.approx(np.linalg.norm(b - M @ x) / np.linalg.norm(b), rel=1e-10)


def test_truncated_solve_books(O):  # test_solver.cpp:83-133
    n = 80
    M = random_matrix(O, n, 83)
    b = O.gaussian_vector(n, 84)
    x, rep = O.solve(O.SparseMatrix.from_dense(M), b, O.SolverConfig(m=10, t=2, k=4, s=60, tol=1e-8, max_restarts=8))
    assert rep.status == "converged"
    assert np.linalg.norm(b - M @ x) <= 1e-8 * np.linalg.norm(b) * (1 + 1e-10)
    for cs in rep.cycle_stats:
        assert cs["basis_cond"] >= 1.0


def test_degenerate_divergence_budget_determinism(O):  # test_solver.cpp:180-259
    n = 30
    A = O.SparseMatrix.from_dense(random_matrix(O, n, 88))
    x, rep = O.solve(A, np.zeros(n), O.SolverConfig(m=5, t=2, k=0, s=12))
    assert rep.status == "converged" and rep.iterations == 0 and rep.counters["matvecs"] == 0
    x, rep = O.solve(O.SparseMatrix.from_dense(2.5 * np.eye(n)), O.gaussian_vector(n, 89), O.SolverConfig(m=5, t=2, k=0, s=12))
    assert rep.status == "converged" and rep.iterations == 1
    C = np.zeros((40, 40))
    for j in range(40):
        C[(j + 1) % 40, j] = 1.0
    b = np.zeros(40)
    b[0] = 1.0
    x, rep = O.solve(O.SparseMatrix.from_dense(C), b, O.SolverConfig(m=5, t=5, k=0, s=40, tol=1e-8, max_restarts=6),
                     sketch=O.SketchOperator.identity(40))
    assert rep.status == "diverged" and rep.cycles == 1
    A = O.SparseMatrix.from_dense(random_matrix(O, 100, 90))
    x, rep = O.solve(A, O.gaussian_vector(100, 91), O.SolverConfig(m=5, t=2, k=0, s=30, tol=1e-13, max_restarts=1))
    assert rep.status == "max_restarts" and rep.iterations == 5
    A = O.SparseMatrix.from_dense(random_matrix(O, 70, 92))
    b = O.gaussian_vector(70, 93)
    c = O.SolverConfig(m=8, t=2, k=3, s=44, tol=1e-8)
    assert np.array_equal(O.solve(A, b, c)[0], O.solve(A, b, c)[0])


def test_config_validation(O):  # test_solver.cpp:261-302
    A = O.SparseMatrix.from_dense(random_matrix(O, 30, 94))
    b = O.gaussian_vector(30, 95)
    for mut in [dict(m=0), dict(t=0), dict(k=5), dict(k=-1), dict(tol=0.0), dict(tol=1.0), dict(safety_init=0.5),
                dict(max_restarts=0), dict(s=13)]:
        kw = dict(m=5, t=2, k=2, s=20)
        kw.update(mut)
        with pytest.raises(ValueError):
            O.solve(A, b, O.SolverConfig(**kw))


def test_sequence_recycling_cuts_iterations(O):  # test_sequence.cpp:46-74
    M = O.gen_neumann(20, 0.05)
    rhs = [O.gaussian_vector(400, 1234 + i) for i in range(3)]
    cfg = O.SolverConfig(m=30, t=2, k=8, s=300, tol=1e-8)
    xs, reps = O.solve_sequence([M] * 3, rhs, cfg, tols=[1e-8] * 3, shared_matrix=True)
    assert all(r.status == "converged" for r in reps)
    assert reps[1].iterations < reps[0].iterations and reps[2].iterations <= reps[1].iterations


# ---------------------------------------------------------------- baseline
# baseline.hpp:51-216 (classical restarted GMRES, the comparison point)

def _dense_gmres_residuals(A, b, m):
    """Minimal residual over K_p(A, b) for p = 1..m (Arnoldi in numpy, then
    a dense least-squares solve per p) — an independent restatement."""
    n = len(b)
    V = np.zeros((n, m + 1))
    H = np.zeros((m + 1, m))
    beta = np.linalg.norm(b)
    V[:, 0] = b / beta
    out = []
    for q in range(m):
        w = A @ V[:, q]
        for _ in range(2):
            h = V[:, :q + 1].T @ w
            w -= V[:, :q + 1] @ h
            H[:q + 1, q] += h
        H[q + 1, q] = np.linalg.norm(w)
        V[:, q + 1] = w / H[q + 1, q]
        e1 = np.zeros(q + 2)
        e1[0] = beta
        y = np.linalg.lstsq(H[:q + 2, :q + 1], e1, rcond=None)[0]
        out.append(np.linalg.norm(e1 - H[:q + 2, :q + 1] @ y))
    return np.array(out)


def test_baseline_estimates_are_minimal_residuals(O):
    A = random_matrix(O, 60, 41)
    b = O.gaussian_vector(60, 42)
    M = O.SparseMatrix.from_dense(A)
    x, rep = O.baseline_gmres(M, b, m=12, tol=1e-14, max_restarts=1)
    est = np.array([v for _, v in rep.sketched_residuals])
    np.testing.assert_allclose(est, _dense_gmres_residuals(A, b, 12), rtol=1e-7, atol=1e-15 * np.linalg.norm(b))
    assert rep.status == "max_restarts" and rep.iterations == 12 and rep.cycles == 1
    # one verification product per cycle; the verified residual is b - A x
    assert rep.true_residuals[0][0] == 12
    assert rep.true_residuals[0][1] == pytest.approx(np.linalg.norm(b - A @ x), rel=1e-9)
    assert rep.true_residuals[0][1] == pytest.approx(est[-1], rel=1e-8)


def test_baseline_counters_closed_form(O):
    # 1 (||b||) + per cycle: 1 (beta) + sum_q (q+1 dots + ||w||) + 1 (verification)
    M = O.gen_convdiff(20, -20.0)
    b = O.gaussian_vector(400, 3)
    x, rep = O.baseline_gmres(M, b, m=10, tol=1e-12, max_restarts=3)
    assert rep.status == "max_restarts" and rep.iterations == 30
    assert rep.counters == {"matvecs": 30 + 3, "inner_products": 1 + 3 * (1 + sum(q + 2 for q in range(10)) + 1),
                            "sketch_applies": 0}
    assert len(rep.sketched_residuals) == 30 and [i for i, _ in rep.true_residuals] == [10, 20, 30]


def test_baseline_converges_and_restarts(O):
    M = O.gen_convdiff(30, -10.0)
    b = O.gaussian_vector(900, 5)
    x, rep = O.baseline_gmres(M, b, m=40, tol=1e-8, max_restarts=30)
    off, col, val = M.csr()
    import scipy.sparse as sp
    A = sp.csr_matrix((val, col, off), shape=(900, 900))
    assert rep.status == "converged" and rep.cycles > 1
    assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) < 1e-8
    assert rep.final_relative_residual == pytest.approx(rep.true_residuals[-1][1] / rep.rhs_norm)


def test_baseline_edge_cases(O):
    n = 30
    I3 = O.SparseMatrix.from_dense(3.0 * np.eye(n))
    b = O.gaussian_vector(n, 9)
    x, rep = O.baseline_gmres(I3, b, m=5, tol=1e-10)  # A = cI: one step
    assert rep.status == "converged" and rep.iterations == 1
    np.testing.assert_allclose(x, b / 3.0, rtol=1e-14)
    x, rep = O.baseline_gmres(I3, np.zeros(n), m=5, tol=1e-10)  # zero rhs: no step
    assert rep.status == "converged" and rep.iterations == 0 and rep.cycles == 0
    assert not np.any(x)
    # cyclic shift, b = e_0: the residual cannot drop before step n -> diverged
    P = np.roll(np.eye(n), 1, axis=0)
    e0 = np.zeros(n)
    e0[0] = 1.0
    x, rep = O.baseline_gmres(O.SparseMatrix.from_dense(P), e0, m=10, tol=1e-8, max_restarts=5)
    assert rep.status == "diverged" and rep.iterations == 10
    assert rep.notes == ["cycle 1: residual estimate improved by less than 1% over a full cycle"]
    # x0 = exact solution: beta == 0 at the first cycle
    x, rep = O.baseline_gmres(O.SparseMatrix.from_dense(np.eye(n)), b, m=5, tol=1e-10, x0=b)
    assert rep.status == "converged" and rep.iterations == 0 and rep.counters["matvecs"] == 1
    with pytest.raises(ValueError):
        O.baseline_gmres(I3, b, m=0)
    with pytest.raises(ValueError):
        O.baseline_gmres(I3, b, tol=1.0)


def test_complex_oracle_identity_sketch_is_dense_complex_gmres(O):
    """Pins the complex GMRES-SDR oracle (skrylov_oracle_complex.hpp; no
    reference code exists for complex scalars): with the identity
    sketch, full window and k = 0, every per-step sketched residual equals the
    residual of dense complex GMRES on the same Krylov space (the complex
    analogue of test_solver.cpp:38-81)."""
    rng = np.random.default_rng(0)
    n, m = 40, 12
    M = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)) + n * (1 + 0.5j) * np.eye(n)
    A = O.ZSparseMatrix(n, np.arange(0, n * n + 1, n), np.tile(np.arange(n), n), M.reshape(-1))
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert np.abs(A.apply(x) - M @ x).max() <= 1e-12 * np.abs(M @ x).max()
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    cfg = O.SolverConfig(m=m, t=m, k=0, s=n, tol=1e-10, max_restarts=1)
    xs, rep = O.zsolve(A, b, cfg, O.SketchOperator.identity(n))
    K = np.column_stack([np.linalg.matrix_power(M, i) @ b for i in range(m)])
    for it, sres in rep.sketched_residuals:
        Q, _ = np.linalg.qr(K[:, :it])
        y = np.linalg.lstsq(M @ Q, b, rcond=None)[0]
        assert sres == pytest.approx(np.linalg.norm(b - M @ Q @ y), rel=1e-8)
    assert rep.counters["matvecs"] == m + 1 and rep.counters["sketch_applies"] == m + 1


def test_complex_oracle_recycling_and_counters(O):
    """Complex GMRES-SDR with a real SRDCT sketch on Re / Im and a recycle
    space carried to a second right-hand side: converges, the carried space
    cuts iterations, an exact refresh costs k matvecs + k sketches."""
    rng = np.random.default_rng(1)
    n = 600
    off, col, val = [0], [], []
    for r in range(n):
        for c, v in ((r - 1, -1.0 + 0.3j), (r, 4.0 + 0.5j), (r + 1, -1.2 - 0.2j), (r + 7, 0.4j)):
            if 0 <= c < n:
                col.append(c)
                val.append(v)
        off.append(len(col))
    A = O.ZSparseMatrix(n, off, col, val)
    S = O.SketchOperator.subsampled_dct(n, 60, 0x5EED)
    cfg = O.SolverConfig(m=20, t=2, k=5, s=60, tol=1e-10, max_restarts=30)
    sp = O.ZRecycleSpace()
    b1 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x1, r1 = O.zsolve(A, b1, cfg, S, space=sp)
    assert r1.status == "converged" and sp.dim == 5
    dense = np.zeros((n, n), dtype=complex)
    for r in range(n):
        for p in range(off[r], off[r + 1]):
            dense[r, col[p]] = val[p]
    assert np.linalg.norm(dense @ x1 - b1) <= 1e-10 * np.linalg.norm(b1) * 1.01
    cnt = sp.refresh(A, S)
    assert cnt == dict(matvecs=5, inner_products=0, sketch_applies=5)
    x2, r2 = O.zsolve(A, b1 + 0.01 * (rng.standard_normal(n) + 1j * rng.standard_normal(n)), cfg, S, space=sp)
    assert r2.status == "converged" and r2.iterations < r1.iterations
