"""Cases run by tests/test_gpu_fused_step.py in a subprocess with
SDR_FUSE_STEP=1 (the opt-in path; the switch is read once per process).

KF — one launch per Arnoldi step (fused_step.cu): the update + sparse-sign
sketch of step j and the SpMV + window dots of step j+1 in a single pass, the
SpMV warps trailing the update front chunk by chunk.

Parity bar as for the two-kernel step: H, SV, SAV and V of sdr_krylov_run
within 1e-12 of the oracle's literal truncated Arnoldi (arnoldi.hpp:82-119),
on sizes with one chunk and with many (the chunk waits), stencil reaches
larger than a chunk, t = 1..3; runs are bitwise reproducible; solves with
C5's parameters equal the oracle's (status, cycles, iterations, counters).
"""
import numpy as np
import pytest

from tests.test_gpu_parity import krylov, rel, to_both

pytestmark = pytest.mark.gpu


def conv3d(sk, O, n, beta=(200.0, 100.0, 50.0)):
    off, col, val = sk.gen_convdiff3d(n, *beta)
    N = n ** 3
    return to_both(sk, O, off, col, val, N, N)


def banded(sk, O, N, offsets, seed):
    rows, cols = [], []
    for d in offsets:
        r = np.arange(max(0, -d), min(N, N - d))
        rows.append(r)
        cols.append(r + d)
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = O.gaussian_vector(len(r), seed) + np.where(r == c, 8.0, 0.0)
    return sk.SparseMatrix.from_triplets(N, N, r, c, v), O.SparseMatrix.from_triplets(N, N, r, c, v)


def fused_launches(sk, A, S, r0, t, steps):
    ctx = sk.default_context()
    ctx.set_timing(True)
    ctx.timing_reset()
    try:
        g = krylov(sk, A, S, r0, t, steps)
        n, _ = ctx.timing("fused_step")
    finally:
        ctx.set_timing(False)
    return g, n


def check(g, o, steps):
    assert g["j"] == o.j == steps
    assert g["counters"] == tuple(o.counters)
    assert rel(g["H"], o.H) <= 1e-12
    assert rel(g["SV"], o.SV) <= 1e-12
    assert rel(g["SAV"], o.SAV) <= 1e-12
    assert rel(g["V"], o.V) <= 1e-12


@pytest.mark.parametrize("n", [24, 64, 100])
@pytest.mark.parametrize("t", [1, 2, 3])
def test_fused_step_matches_oracle_convdiff3d(sk, O, n, t):
    """3-D 7-point operators (SELL-DIA): 24^3 fits one chunk, 64^3 and 100^3
    (1 M rows, 2.2 chunks of a 444-CTA grid) make the SpMV warps wait on the
    update front; the plane reach (n^2 rows) spans several tiles."""
    A, Ao = conv3d(sk, O, n)
    N = n ** 3
    S, So = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8), O.SketchOperator.sparse_sign(N, 120, 0x5EED, 8)
    r0 = O.gaussian_vector(N, 3)
    steps = 10
    g, nf = fused_launches(sk, A, S, r0, t, steps)
    assert nf == steps - 1, nf  # K1(0), then one fused launch per step, the last step K2s alone
    check(g, O.run_arnoldi(Ao, r0, So, t, steps), steps)


@pytest.mark.parametrize("N,offsets", [(1 << 21, (-250001, -1, 0, 1, 249999)),
                                       (700001, (-5, -1, 0, 2, 250000)),
                                       (513, (-7, -1, 0, 1, 3))])
def test_fused_step_long_reach_and_ragged(sk, O, N, offsets):
    """A stencil reach longer than a chunk (250 k rows), an odd length with a
    partial last tile, and the smallest eligible length (one tile + 1 row)."""
    A, Ao = banded(sk, O, N, offsets, 11)
    S, So = sk.SketchOperator.sparse_sign(N, 100, 0x5EED, 8), O.SketchOperator.sparse_sign(N, 100, 0x5EED, 8)
    r0 = O.gaussian_vector(N, 5)
    steps = 6
    g, nf = fused_launches(sk, A, S, r0, 2, steps)
    assert nf == steps - 1, nf
    check(g, O.run_arnoldi(Ao, r0, So, 2, steps), steps)


def test_fused_step_bitwise_reproducible(sk, O):
    A, _ = conv3d(sk, O, 64)
    N = 64 ** 3
    S = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8)
    r0 = O.gaussian_vector(N, 3)
    a = krylov(sk, A, S, r0, 2, 12)
    b = krylov(sk, A, S, r0, 2, 12)
    for k in ("H", "SV", "SAV", "V"):
        assert np.array_equal(a[k], b[k]), k


def test_fused_step_c5_parameters_solve_matches_oracle(sk, O):
    """C5's solver parameters at 64^3 (sparse sign, m=50 k=10 t=2 s=120, tol
    1e-7): every step but a cycle's first and last is a fused launch."""
    n = 64
    A, Ao = conv3d(sk, O, n)
    N = n ** 3
    S, So = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8), O.SketchOperator.sparse_sign(N, 120, 0x5EED, 8)
    b = O.gaussian_vector(N, 3)
    cfg = dict(m=50, k=10, t=2, s=120, tol=1e-7, max_restarts=100)
    ctx = sk.default_context()
    ctx.set_timing(True)
    ctx.timing_reset()
    try:
        r = sk.solve(A, b, sk.SolverConfig(**cfg), sketch=S)
        nf, _ = ctx.timing("fused_step")
    finally:
        ctx.set_timing(False)
    xo, ro = O.solve(Ao, b, O.SolverConfig(**cfg), sketch=So)
    assert nf > 0
    assert r.report.status == ro.status == "converged"
    assert abs(r.report.iterations - ro.iterations) <= max(1, 0.02 * ro.iterations)
    if r.report.iterations == ro.iterations:
        assert r.report.cycles == ro.cycles
        assert r.report.counters == ro.counters
    assert r.report.final_relative_residual < 1e-7
    assert rel(r.x, xo) <= 1e-5
