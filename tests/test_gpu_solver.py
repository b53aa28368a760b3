"""GPU solver parity: sdr_solve / sdr_solve_sequence against the CPU oracle
and the reference's solver / sequence properties (test_solver.cpp,
test_sequence.cpp, acceptance.cpp criteria 1 and 6)."""
import numpy as np
import pytest

from tests.test_gpu_parity import random_matrix, rel

pytestmark = pytest.mark.gpu


def both(sk, O, M):
    return sk.SparseMatrix.from_dense(M), O.SparseMatrix.from_dense(M)


def cfgs(sk, O, **kw):
    return sk.SolverConfig(**kw), O.SolverConfig(**kw)


def assert_same_solve(g, o, iters_tol=0.0):
    assert g.report.status == o[1].status
    if iters_tol == 0.0:
        assert g.report.iterations == o[1].iterations
        assert g.report.cycles == o[1].cycles
        assert g.report.counters == o[1].counters
    else:
        assert abs(g.report.iterations - o[1].iterations) <= max(1, iters_tol * o[1].iterations)


def test_identity_sketch_reproduces_dense_gmres(sk, O):
    n, m = 40, 20
    M = random_matrix(O, n, 81)
    A, Ao = both(sk, O, M)
    b = O.gaussian_vector(n, 82)
    c, co = cfgs(sk, O, m=m, t=m, k=0, s=2 * m, tol=1e-8, safety_init=1.0, max_restarts=2)
    g = sk.solve(A, b, c, sketch=sk.SketchOperator.identity(n))
    o = O.solve(Ao, b, co, sketch=O.SketchOperator.identity(n))
    assert g.report.status == "converged" and g.report.cycles == 1
    assert_same_solve(g, o)
    for (i1, v1), (i2, v2) in zip(g.report.sketched_residuals, o[1].sketched_residuals):
        assert i1 == i2 and abs(v1 - v2) <= 1e-8 * np.linalg.norm(b)
    xr = np.linalg.solve(M, b)
    assert np.linalg.norm(g.x - o[0]) <= 1e-8 * np.linalg.norm(xr)
    assert g.report.final_relative_residual == pytest.approx(np.linalg.norm(b - M @ g.x) / np.linalg.norm(b), rel=1e-10)


def test_truncated_sketched_solve_books(sk, O):
    n = 80
    M = random_matrix(O, n, 83)
    A, Ao = both(sk, O, M)
    b = O.gaussian_vector(n, 84)
    c, co = cfgs(sk, O, m=10, t=2, k=4, s=60, tol=1e-8, max_restarts=8)
    g = sk.solve(A, b, c)
    o = O.solve(Ao, b, co)
    assert g.report.status == "converged"
    assert_same_solve(g, o)
    res = np.linalg.norm(b - M @ g.x)
    assert res <= c.tol * np.linalg.norm(b) * (1 + 1e-10)
    assert g.report.final_relative_residual == pytest.approx(res / np.linalg.norm(b), rel=1e-9)
    idx = 0
    for cs in g.report.cycle_stats:
        prev = np.inf
        for _ in range(cs["steps"]):
            v = g.report.sketched_residuals[idx][1]
            assert v <= prev * (1 + 1e-12)
            prev = v
            idx += 1
        assert cs["basis_cond"] >= 1.0
    safety = 0.0
    for cs in g.report.cycle_stats:
        assert cs["safety_after"] >= safety
        safety = cs["safety_after"]
    assert g.space.dim() >= c.k
    # recycle_consistency_error (recycle.hpp:389-403): SU = S U, SAU = S A U
    S = O.SketchOperator.subsampled_dct(n, c.s, c.sketch_seed)
    U, SU, SAU = g.space.get()
    for q in range(U.shape[1]):
        assert np.linalg.norm(S.apply(U[:, q]) - SU[:, q]) / max(1.0, np.linalg.norm(SU[:, q])) <= 1e-10
        assert np.linalg.norm(S.apply(M @ U[:, q]) - SAU[:, q]) / max(1.0, np.linalg.norm(SAU[:, q])) <= 1e-10
        assert np.linalg.norm(U[:, q]) == pytest.approx(1.0, abs=1e-13)


def test_degenerate_rhs(sk, O):
    n = 30
    A = sk.SparseMatrix.from_dense(random_matrix(O, n, 88))
    c = sk.SolverConfig(m=5, t=2, k=0, s=12)
    z = sk.solve(A, np.zeros(n), c)
    assert z.report.status == "converged" and z.report.iterations == 0
    assert z.report.counters["matvecs"] == 0 and np.linalg.norm(z.x) == 0.0
    assert z.report.final_relative_residual == 0.0
    Cm = sk.SparseMatrix.from_dense(2.5 * np.eye(n))
    b = O.gaussian_vector(n, 89)
    e = sk.solve(Cm, b, c)
    assert e.report.status == "converged" and e.report.iterations == 1
    assert np.linalg.norm(e.x - b / 2.5) <= 1e-12 * np.linalg.norm(b)


def test_stagnation_is_divergence(sk, O):
    n = 40
    M = np.zeros((n, n))
    for j in range(n):
        M[(j + 1) % n, j] = 1.0
    b = np.zeros(n)
    b[0] = 1.0
    c = sk.SolverConfig(m=5, t=5, k=0, s=n, tol=1e-8, max_restarts=6)
    r = sk.solve(sk.SparseMatrix.from_dense(M), b, c, sketch=sk.SketchOperator.identity(n))
    assert r.report.status == "diverged" and r.report.cycles == 1 and r.report.notes


def test_restart_budget(sk, O):
    n = 100
    A = sk.SparseMatrix.from_dense(random_matrix(O, n, 90))
    r = sk.solve(A, O.gaussian_vector(n, 91), sk.SolverConfig(m=5, t=2, k=0, s=30, tol=1e-13, max_restarts=1))
    assert r.report.status == "max_restarts" and r.report.cycles == 1 and r.report.iterations == 5


def test_bitwise_determinism(sk, O):
    n = 70
    A = sk.SparseMatrix.from_dense(random_matrix(O, n, 92))
    b = O.gaussian_vector(n, 93)
    c = sk.SolverConfig(m=8, t=2, k=3, s=44, tol=1e-8)
    r1, r2 = sk.solve(A, b, c), sk.solve(A, b, c)
    assert r1.report.status == r2.report.status and r1.report.iterations == r2.report.iterations
    assert np.array_equal(r1.x, r2.x)


def test_config_validation_and_shapes(sk, O):
    n = 30
    M = random_matrix(O, n, 94)
    A = sk.SparseMatrix.from_dense(M)
    b = O.gaussian_vector(n, 95)
    for mut in [dict(m=0), dict(t=0), dict(k=5), dict(k=-1), dict(tol=0.0), dict(tol=1.0), dict(safety_init=0.5),
                dict(max_restarts=0), dict(s=13)]:
        kw = dict(m=5, t=2, k=2, s=20)
        kw.update(mut)
        with pytest.raises(ValueError):
            sk.solve(A, b, sk.SolverConfig(**kw))
    ok = sk.SolverConfig(m=5, t=2, k=2, s=20)
    with pytest.raises(ValueError):
        sk.solve(A, np.zeros(n + 1), ok)
    with pytest.raises(ValueError):
        sk.solve(A, b, ok, sketch=sk.SketchOperator.subsampled_dct(n - 1, 20, 1))
    with pytest.raises(ValueError):
        sk.solve(A, b, ok, x0=np.zeros(n - 1))
    g = O.gaussian_vector(n, 96)
    w = sk.solve(A, b, ok, x0=g)
    assert w.report.status == "converged"
    assert np.linalg.norm(b - M @ w.x) <= ok.tol * np.linalg.norm(b) * (1 + 1e-10)


def test_c1_problem_matches_oracle(sk, O):
    """BASELINE config C1: A = -gen_convdiff(100, -50), b ~ N(0,1) seed 0 normalised,
    m=50, k=10, t=2, s=120, tol 1e-8 — SRDCT (reference sketch) and sparse sign."""
    off, col, val = O.gen_convdiff(100, -50.0).csr()
    A = sk.SparseMatrix(10000, 10000, off, col, -val)
    Ao = O.SparseMatrix.from_csr(10000, 10000, off, col, -val)
    b = O.gaussian_vector(10000, 0)
    b /= np.linalg.norm(b)
    c, co = cfgs(sk, O, m=50, k=10, t=2, s=120, tol=1e-8, max_restarts=40)
    g = sk.solve(A, b, c)
    o = O.solve(Ao, b, co)
    assert_same_solve(g, o, iters_tol=0.02)
    assert g.report.final_relative_residual <= 1e-8 or g.report.status != "converged"
    gs = sk.solve(A, b, c, sketch=sk.SketchOperator.sparse_sign(10000, 120, 0x5EED, 8))
    os_ = O.solve(Ao, b, co, sketch=O.SketchOperator.sparse_sign(10000, 120, 0x5EED, 8))
    assert_same_solve(gs, os_, iters_tol=0.02)


def test_sequence_recycling_cuts_iterations(sk, O):
    """test_sequence.cpp:46-74: neumann_sequence(20, 0.05, 3, 1234, 1e-8), m=30 t=2 k=8 s=300."""
    M = O.gen_neumann(20, 0.05).dense()
    A, Ao = sk.SparseMatrix.from_dense(M), O.SparseMatrix.from_dense(M)
    rhs = [O.gaussian_vector(400, 1234 + i) for i in range(3)]
    c, co = cfgs(sk, O, m=30, t=2, k=8, s=300, tol=1e-8, max_restarts=10)
    res = sk.solve_sequence([sk.ProblemInstance(A, b, target_tol=1e-8) for b in rhs], c, shared_matrix=True)
    xs, reps = O.solve_sequence([Ao] * 3, rhs, co, tols=[1e-8] * 3, shared_matrix=True)
    for i, (gr, orr) in enumerate(zip(res.reports, reps)):
        assert gr.status == orr.status == "converged"
        assert abs(gr.iterations - orr.iterations) <= max(1, 0.02 * orr.iterations)
        assert np.linalg.norm(rhs[i] - M @ res.solutions[i]) <= 1e-8 * np.linalg.norm(rhs[i]) * (1 + 1e-10)
    assert res.reports[1].iterations < res.reports[0].iterations
    assert res.reports[2].iterations <= res.reports[1].iterations
    assert res.space.dim() >= 8 and res.space.provenance == "reused"
    warm = sk.solve_sequence([sk.ProblemInstance(A, O.gaussian_vector(400, 9876), target_tol=1e-8)], c,
                             initial_space=res.space, shared_matrix=True)
    assert warm.reports[0].status == "converged"
    assert warm.reports[0].iterations < res.reports[0].iterations


def test_sequence_variants_match_oracle(sk, O):
    """test_sequence.cpp:105-147: exact refresh costs k matvecs + k sketches
    charged to the changed system; reuse on a changed matrix leaves a note."""
    n = 400
    g = 20
    M1 = O.gen_neumann(g, 0.5).dense()
    M2 = O.gen_neumann(g, 0.7).dense()
    A1, A2 = sk.SparseMatrix.from_dense(M1), sk.SparseMatrix.from_dense(M2)
    A1o, A2o = O.SparseMatrix.from_dense(M1), O.SparseMatrix.from_dense(M2)
    rhs = [O.gaussian_vector(n, 500 + i) for i in range(4)]
    for variant in ("exact", "inexact", "reuse"):
        c, co = cfgs(sk, O, m=30, k=8, t=2, s=80, tol=1e-8, variant=variant)
        probs = [sk.ProblemInstance(A1, rhs[0]), sk.ProblemInstance(A1, rhs[1]), sk.ProblemInstance(A2, rhs[2]),
                 sk.ProblemInstance(A2, rhs[3])]
        res = sk.solve_sequence(probs, c)
        xs, reps = O.solve_sequence([A1o, A1o, A2o, A2o], rhs, co)
        for gr, orr in zip(res.reports, reps):
            assert gr.status == orr.status
            assert abs(gr.iterations - orr.iterations) <= max(1, 0.02 * orr.iterations)
            assert gr.counters["matvecs"] - gr.iterations == orr.counters["matvecs"] - orr.iterations
            assert gr.notes[-1:] == orr.notes[-1:] or variant != "reuse"
        if variant == "exact":
            # the changed system pays k matvecs + k sketches for the refresh
            k_carried = res.reports[2].counters["sketch_applies"] - (res.reports[2].iterations + res.reports[2].cycles)
            assert k_carried == reps[2].counters["sketch_applies"] - (reps[2].iterations + reps[2].cycles)


def test_sequence_failure_isolation_and_empty(sk, O):
    n = 50
    A = sk.SparseMatrix.from_dense(random_matrix(O, n, 5))
    B = sk.SparseMatrix.from_dense(random_matrix(O, n + 1, 6))
    c = sk.SolverConfig(m=10, k=3, t=2, s=30, tol=1e-8)
    res = sk.solve_sequence([sk.ProblemInstance(A, O.gaussian_vector(n, 1)),
                             sk.ProblemInstance(B, O.gaussian_vector(n + 1, 2)),
                             sk.ProblemInstance(A, O.gaussian_vector(n, 3))], c)
    assert res.reports[0].status == "converged"
    assert res.reports[1].error and "aborted" in res.reports[1].notes[-1]
    assert res.reports[2].status == "converged"
    assert sk.solve_sequence([], c).reports == []


def test_c4_real_equivalent_small_lattice_matches_oracle(sk, O):
    """BASELINE C4's operator (complex 4-D lattice) at 4^4 sites in its
    real-equivalent form (tools/c4_problem.py): GPU solve == oracle solve."""
    from tools.c4_problem import c4_csr
    off, col, val = c4_csr((4, 4, 4, 4), m0=-0.8, seed=2, uniform=O.uniform_stream)
    n2 = len(off) - 1
    A = sk.SparseMatrix(n2, n2, off, col, val)
    Ao = O.SparseMatrix.from_csr(n2, n2, off, col, val)
    b = O.gaussian_vector(n2, 4)
    c, co = cfgs(sk, O, m=20, k=6, t=3, s=60, tol=1e-8, max_restarts=30)
    g = sk.solve(A, b, c)
    o = O.solve(Ao, b, co)
    assert_same_solve(g, o, iters_tol=0.02)
    assert g.report.status == "converged"
    # the interleaved solution is the complex solution of (4 + m0) x + sum couplings = b
    z = g.x[0::2] + 1j * g.x[1::2]
    Ac = (O.SparseMatrix.from_csr(n2, n2, off, col, val).dense())
    Acx = Ac[0::2, 0::2] + 1j * Ac[1::2, 0::2]
    bc = b[0::2] + 1j * b[1::2]
    assert np.linalg.norm(Acx @ z - bc) <= 1e-7 * np.linalg.norm(bc)


def test_distributed_pipeline_on_one_rank(sk, O):
    """The multi-GPU code path (NCCL halo plans and allreduces, last-CTA folds,
    coefficients formed after the allreduce, fold kernel + allreduce of the B
    record) run on a one-rank NCCL communicator: same solve as the one-GPU
    deferred pipeline and the oracle."""
    cfg = sk.SolverConfig(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=20)
    n = 24
    dctx = sk.Context(0, 0, 1, sk.Context.nccl_unique_id())
    Ad = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0, ctx=dctx)
    A1 = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0)
    b = O.gaussian_vector(n ** 3, 1)
    gd = sk.solve(Ad, b, cfg, space=sk.RecycleSpace(dctx),
                  sketch=sk.SketchOperator.subsampled_dct(n ** 3, 80, cfg.sketch_seed, ctx=dctx))
    g1 = sk.solve(A1, b, cfg)
    Ao = O.gen_convdiff3d(n, 100.0, 50.0, 25.0)
    o = O.solve(Ao, b, O.SolverConfig(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=20))
    assert gd.report.status == g1.report.status == o[1].status
    assert gd.report.iterations == g1.report.iterations
    assert abs(gd.report.iterations - o[1].iterations) <= max(1, 0.02 * o[1].iterations)
    for (i1, r1), (i2, r2) in zip(gd.report.true_residuals, g1.report.true_residuals):
        assert i1 == i2 and r1 == pytest.approx(r2, rel=1e-8)
    assert np.linalg.norm(gd.x - g1.x) <= 1e-9 * np.linalg.norm(g1.x)


def test_distributed_split_k1_matches(sk, O):
    """The several-rank K1 split (interior slices beside the halo transfer,
    boundary slices after it, partials folded over both launches) forced on a
    one-rank communicator (SDR_K1_SPLIT=force, a fresh process): same solve."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, ".")
import paper_2311_14206_b200 as sk
from oracle import pyoracle as O
n = 24
cfg = sk.SolverConfig(m=30, k=8, t=2, s=80, tol=1e-8, max_restarts=20)
ctx = sk.Context(0, 0, 1, sk.Context.nccl_unique_id())
A = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0, ctx=ctx)
b = O.gaussian_vector(n ** 3, 1)
r = sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=sk.SketchOperator.subsampled_dct(n ** 3, 80, cfg.sketch_seed, ctx=ctx))
print(json.dumps(dict(it=r.report.iterations, st=r.report.status, res=[v for _, v in r.report.true_residuals],
                      x=np.asarray(r.x).tolist())))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("0", "force"):
        env = dict(os.environ, SDR_K1_SPLIT=mode)
        p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        outs[mode] = json.loads(p.stdout.strip().splitlines()[-1])
    a, f = outs["0"], outs["force"]
    assert a["st"] == f["st"] and a["it"] == f["it"]
    np.testing.assert_allclose(f["res"], a["res"], rtol=1e-8)
    np.testing.assert_allclose(f["x"], a["x"], rtol=1e-8, atol=1e-10 * np.linalg.norm(a["x"]))


@pytest.mark.parametrize("t", [1, 2, 3, 4, 6])
@pytest.mark.parametrize("k", [0, 6])
@pytest.mark.parametrize("sketch", ["srdct", "sparse"])
def test_config_sweep_matches_oracle(sk, O, t, k, sketch):
    """Window t (fused update+SRDCT up to t = 4, the unfused path beyond),
    deflation on / off, both sketches, on a 32^3 convection-diffusion system
    (deferred step pipeline eligible): same status, iterations within 2 %,
    identical books when the iteration counts agree."""
    n = 32
    off, col, val = sk.gen_convdiff3d(n, 60.0, 30.0, 15.0)
    N = n ** 3
    A = sk.SparseMatrix(N, N, off, col, val)
    Ao = O.SparseMatrix.from_csr(N, N, off, col, val)
    b = O.gaussian_vector(N, 7)
    kw = dict(m=30, t=t, k=k, s=80, tol=1e-8, max_restarts=30)
    if sketch == "srdct":
        S, So = sk.SketchOperator.subsampled_dct(N, 80, 0x5EED), O.SketchOperator.subsampled_dct(N, 80, 0x5EED)
    else:
        S, So = sk.SketchOperator.sparse_sign(N, 80, 0x5EED, 8), O.SketchOperator.sparse_sign(N, 80, 0x5EED, 8)
    g = sk.solve(A, b, sk.SolverConfig(**kw), sketch=S)
    o = O.solve(Ao, b, O.SolverConfig(**kw), sketch=So)
    assert_same_solve(g, o, iters_tol=0.02)
    if g.report.iterations == o[1].iterations:
        assert g.report.counters == o[1].counters
    if o[1].status == "converged":
        assert np.linalg.norm(b - Ao.apply(g.x)) <= 1e-8 * np.linalg.norm(b) * (1 + 1e-9)


def test_nonzero_x0_matches_oracle(sk, O):
    """solver.hpp:307-316: r0 = b - A x0 with one extra product booked."""
    n = 32
    off, col, val = sk.gen_convdiff3d(n, 60.0, 30.0, 15.0)
    N = n ** 3
    A = sk.SparseMatrix(N, N, off, col, val)
    Ao = O.SparseMatrix.from_csr(N, N, off, col, val)
    b = O.gaussian_vector(N, 3)
    x0 = 0.01 * O.gaussian_vector(N, 4)
    kw = dict(m=25, t=2, k=5, s=60, tol=1e-9, max_restarts=30)
    g = sk.solve(A, b, sk.SolverConfig(**kw), x0=x0)
    o = O.solve(Ao, b, O.SolverConfig(**kw), x0=x0)
    assert_same_solve(g, o, iters_tol=0.02)
    if g.report.iterations == o[1].iterations:
        assert g.report.counters == o[1].counters
    assert np.linalg.norm(b - Ao.apply(g.x)) <= 1e-9 * np.linalg.norm(b) * (1 + 1e-9)


def test_breakdown_status_and_note(sk, O):
    """A lucky breakdown that does not solve the system (b has a component in
    the null space of a singular A) ends the solve as `breakdown` with the
    reference's note (solver.hpp:344-350)."""
    n = 60
    d = np.linspace(1.0, 3.0, n)
    d[-1] = 0.0  # singular
    M = np.diag(d)
    A, Ao = sk.SparseMatrix.from_dense(M), O.SparseMatrix.from_dense(M)
    b = np.zeros(n)
    b[:3] = 1.0
    b[-1] = 1.0  # null-space component: the residual cannot drop below 1
    kw = dict(m=10, t=10, k=0, s=40, tol=1e-8, max_restarts=5)
    g = sk.solve(A, b, sk.SolverConfig(**kw))
    o = O.solve(Ao, b, O.SolverConfig(**kw))
    assert g.report.status == o[1].status == "breakdown"
    assert g.report.iterations == o[1].iterations
    assert g.report.notes == o[1].notes


def test_workspace_reuse_across_operators(sk, O):
    """One context, operators of different sizes / storage forms / windows in
    turn (the cached workspace is re-laid out): every solve equals the first
    solve of the same problem."""
    probs = []
    for n, t, k in ((24, 2, 6), (16, 3, 4), (24, 2, 6), (20, 1, 0), (16, 3, 4)):
        off, col, val = sk.gen_convdiff3d(n, 60.0, 30.0, 15.0)
        N = n ** 3
        probs.append((sk.SparseMatrix(N, N, off, col, val), O.gaussian_vector(N, n), dict(m=20, t=t, k=k, s=60, tol=1e-9,
                                                                                            max_restarts=40)))
    first = {}
    for i, (A, b, kw) in enumerate(probs):
        r = sk.solve(A, b, sk.SolverConfig(**kw))
        key = (A.rows, kw["t"], kw["k"])
        if key in first:
            r0 = first[key]
            assert r.report.iterations == r0.report.iterations
            assert np.array_equal(r.x, r0.x)
        else:
            first[key] = r
        assert r.report.status == "converged"


def test_concurrent_solves_on_separate_contexts(sk, O):
    """Distinct problems on separate contexts may run concurrently (SPEC
    threading contract): two host threads, two contexts, results identical to
    the sequential solves."""
    import threading
    jobs = []
    for n in (24, 20):
        ctx = sk.Context(0)
        off, col, val = sk.gen_convdiff3d(n, 60.0, 30.0, 15.0)
        N = n ** 3
        A = sk.SparseMatrix(N, N, off, col, val, ctx=ctx)
        jobs.append((ctx, A, O.gaussian_vector(N, n), sk.SolverConfig(m=20, t=2, k=5, s=60, tol=1e-9, max_restarts=40)))
    seq = [sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx)) for ctx, A, b, cfg in jobs]
    out = [None, None]

    def run(i):
        ctx, A, b, cfg = jobs[i]
        out[i] = [sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx)) for _ in range(3)]

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(2):
        for r in out[i]:
            assert r.report.iterations == seq[i].report.iterations
            assert np.array_equal(r.x, seq[i].x)


@pytest.mark.parametrize("m,k,t", [(250, 20, 2), (60, 30, 2), (40, 0, 4)])
def test_long_cycles_and_wide_recycle_spaces(sk, O, m, k, t):
    """m = 250 (record / event arrays, 251-column bases), k = 30 (recycle
    product beyond the 24-output kernels: the cuBLAS route), k = 0."""
    n = 20
    off, col, val = sk.gen_convdiff3d(n, 80.0, 40.0, 20.0)
    N = n ** 3
    A = sk.SparseMatrix(N, N, off, col, val)
    Ao = O.SparseMatrix.from_csr(N, N, off, col, val)
    b = O.gaussian_vector(N, 17)
    kw = dict(m=m, t=t, k=k, s=2 * (m + k), tol=1e-10, max_restarts=20)
    g = sk.solve(A, b, sk.SolverConfig(**kw))
    o = O.solve(Ao, b, O.SolverConfig(**kw))
    assert_same_solve(g, o, iters_tol=0.02)
    if o[1].status == "converged":
        assert np.linalg.norm(b - Ao.apply(g.x)) <= 1e-10 * np.linalg.norm(b) * (1 + 1e-9)


@pytest.mark.parametrize("seed,n,m,k,t,kind", [(81, 300, 30, 0, 1, "ss"), (82, 300, 30, 0, 1, "dct"),
                                               (86, 150, 15, 4, 3, "ss")])
def test_failed_verification_continues_the_cycle(sk, O, seed, n, m, k, t, kind):
    """A trigger whose true residual misses the tolerance (safety_init = 1):
    the safety factor ratchets and the same cycle goes on (solver.hpp:199-216)
    — two true-residual checks in one cycle, the first correction discarded.
    Status, iterations, cycles, every true residual and x equal the oracle's."""
    M = random_matrix(O, n, seed)
    A, Ao = both(sk, O, M)
    b = O.gaussian_vector(n, seed + 1000)
    s = 2 * (m + k)
    c, co = cfgs(sk, O, m=m, t=t, k=k, s=s, tol=1e-10, safety_init=1.0, max_restarts=10)
    if kind == "ss":
        S, So = sk.SketchOperator.sparse_sign(n, s, 7, 8), O.SketchOperator.sparse_sign(n, s, 7, 8)
    else:
        S, So = sk.SketchOperator.subsampled_dct(n, s, 7), O.SketchOperator.subsampled_dct(n, s, 7)
    g = sk.solve(A, b, c, sketch=S)
    xo, ro = O.solve(Ao, b, co, sketch=So)
    assert len(ro.true_residuals) > ro.cycles  # the oracle took the failed-check path
    assert g.report.status == ro.status and g.report.iterations == ro.iterations and g.report.cycles == ro.cycles
    assert len(g.report.true_residuals) == len(ro.true_residuals)
    for (i1, v1), (i2, v2) in zip(g.report.true_residuals, ro.true_residuals):
        assert i1 == i2 and v1 == pytest.approx(v2, rel=1e-6, abs=1e-13 * np.linalg.norm(b))
    assert rel(g.x, xo) <= 1e-9
    assert np.linalg.norm(b - M @ g.x) <= 1e-10 * np.linalg.norm(b) * (1 + 1e-6)


def test_sequence_device_resident_rhs_and_solutions(sk, O):
    """solve_sequence with CUDA right-hand sides and caller-owned CUDA solution
    buffers (written in place) gives the host-array run's solutions bit for bit."""
    import torch
    n = 400
    M1, M2 = O.gen_neumann(20, 0.5).dense(), O.gen_neumann(20, 0.7).dense()
    A1, A2 = sk.SparseMatrix.from_dense(M1), sk.SparseMatrix.from_dense(M2)
    rhs = [O.gaussian_vector(n, 700 + i) for i in range(3)]
    c, _ = cfgs(sk, O, m=30, k=8, t=2, s=80, tol=1e-8, variant="exact")
    host = sk.solve_sequence([sk.ProblemInstance(A1, rhs[0]), sk.ProblemInstance(A2, rhs[1]),
                              sk.ProblemInstance(A2, rhs[2])], c)
    outs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    dev = sk.solve_sequence([sk.ProblemInstance(A, torch.from_numpy(b).cuda())
                             for A, b in zip((A1, A2, A2), rhs)], c, outs=outs)
    for i in range(3):
        assert dev.solutions[i] is outs[i]
        assert dev.reports[i].iterations == host.reports[i].iterations
        assert np.array_equal(outs[i].cpu().numpy(), host.solutions[i])
    with pytest.raises(ValueError):
        sk.solve_sequence([sk.ProblemInstance(A1, rhs[0])], c, outs=[np.zeros(n - 1)])


def test_exact_refresh_at_c3_size_matches_per_column_sketches(sk, O):
    """refresh_for_new_matrix (recycle.hpp:297-318) at C3's size (1024^2,
    SRDCT s = 140, k = 20): the k sketches run on concurrent streams into
    their own partials; every SAU column equals S (A u_q) from the one-vector
    apply to 1e-12."""
    n = 1024
    N = n * n
    off, col, val = sk.gen_convdiff2d(n, 100.0, 100.0)
    A = sk.SparseMatrix(N, N, off, col, val)
    off2, col2, val2 = sk.gen_convdiff2d(n, 102.0, 98.0, 0.01)
    A2 = sk.SparseMatrix(N, N, off2, col2, val2)
    S = sk.SketchOperator.subsampled_dct(N, 140, 0x5EED)
    k = 20
    U = np.stack([O.gaussian_vector(N, 900 + q) for q in range(k)], axis=1)
    U /= np.linalg.norm(U, axis=0)
    space = sk.RecycleSpace(A.ctx)
    space.set(U, np.zeros((140, k)), np.zeros((140, k)))
    cnt = space.refresh(A2, S)
    assert cnt["matvecs"] == k and cnt["sketch_applies"] == k
    _, _, SAU = space.get()
    for q in range(k):
        ref = S.apply(A2.apply(U[:, q]))
        assert np.linalg.norm(SAU[:, q] - ref) <= 1e-12 * np.linalg.norm(ref), q
