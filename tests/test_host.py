"""CPU tests of the product's host side and boundary: the C-ABI library loads
and exports every symbol include/sdr_b200.h declares; host generators and
seeded streams are bit-identical to the oracle; the host incremental QR and
harmonic-Ritz extraction match the reference semantics; partition logic.
No compute call here needs a GPU."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest
import scipy.linalg as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ boundary

def test_library_exports_every_header_symbol(sk):
    names = sk._capi.header_symbols()
    assert len(names) >= 60
    out = subprocess.run(["nm", "-D", "--defined-only", sk._capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(sk._lib, n)


def test_library_is_sm100a_and_has_no_cpu_fallback(sk):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sk._capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    v = [C.c_int() for _ in range(3)]
    assert sk._lib.sdr_version(*[C.byref(x) for x in v]) == 0


def test_compute_without_gpu_fails_loudly(sk):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(sk.CudaError):
        sk.Context(0)


def test_config_defaults_and_validation(sk):
    cfg = sk._capi.sdr_config()
    assert sk._lib.sdr_config_default(C.byref(cfg)) == 0
    assert (cfg.m, cfg.t, cfg.k, cfg.s, cfg.tol, cfg.safety_init, cfg.max_restarts, cfg.sketch_seed) == (
        100, 2, 20, 0, 1e-6, 1.4, 10, 0x5EED)
    with pytest.raises(ValueError, match="sketch size s = 0 is below 2 \\(m \\+ k\\) = 240"):
        sk.SolverConfig().validate()
    sk.SolverConfig(s=240).validate()
    with pytest.raises(ValueError, match="need 0 <= k < m"):
        sk.SolverConfig(m=5, k=5, s=100).validate()


# ------------------------------------------------------------ seeded streams

def test_gaussian_vector_bit_exact(sk, O):
    for seed in (0, 1, 3, 0x5EED):
        assert np.array_equal(sk.gaussian_vector(1001, seed), O.gaussian_vector(1001, seed))


@pytest.mark.parametrize("n,s,seed", [(200, 48, 31), (10000, 120, 0x5EED), (2 ** 21, 240, 0x5EED), (65537, 300, 9)])
def test_srdct_indices_bit_exact(sk, O, n, s, seed):
    rows, signs = sk.srdct_indices(n, s, seed)
    So = O.SketchOperator.subsampled_dct(n, s, seed)
    assert np.array_equal(rows, So.rows())
    assert np.array_equal(signs, So.signs())


def test_uniform_stream_bit_exact(sk, O):
    assert np.array_equal(sk.uniform_stream(0x3100, 1000), O.uniform_stream(0x3100, 1000))


def test_sparse_sign_entries_bit_exact(sk, O):
    So = O.SketchOperator.sparse_sign(10 ** 6, 120, 0x5EED, 8)
    for j0 in (0, 12345, 10 ** 6 - 64):
        r1, s1 = sk.sparse_sign_entries(120, 0x5EED, 8, j0, 64)
        r2, s2 = So.sparse_entries(j0, 64, 8)
        assert np.array_equal(r1, r2) and np.array_equal(s1, s2)


# ---------------------------------------------------------------- generators

def test_generators_bit_exact_with_oracle(sk, O):
    off, col, val = sk.gen_convdiff(100, -50.0)
    o2, c2, v2 = O.gen_convdiff(100, -50.0).csr()
    assert np.array_equal(off, o2) and np.array_equal(col, c2) and np.array_equal(val, v2)
    rel = 1e-3 * (2 * O.uniform_stream(0x3101, 32 * 32) - 1)
    a = sk.gen_convdiff2d(32, 102.0, 98.0, 0.01, rel)
    b = O.gen_convdiff2d(32, 102.0, 98.0, 0.01, rel).csr()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    a = sk.gen_convdiff3d(20, 100.0, 50.0, 25.0)
    b = O.gen_convdiff3d(20, 100.0, 50.0, 25.0).csr()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_3d_slab_generator_matches_full_rows(sk):
    n = 12
    off, col, val = sk.gen_convdiff3d(n, 100.0, 50.0, 25.0)
    o3, c3, v3 = sk.gen_convdiff3d(n, 100.0, 50.0, 25.0, z_begin=4, z_end=9)
    r0, r1 = 4 * n * n, 9 * n * n
    assert np.array_equal(c3, col[off[r0]:off[r1]]) and np.array_equal(v3, val[off[r0]:off[r1]])
    assert np.array_equal(o3, off[r0:r1 + 1] - off[r0])


def test_zero_coefficients_dropped_like_from_triplets(sk, O):
    # beta chosen so -h2 + c == 0 on +x: from_triplets drops exact zeros (sparse.hpp:66)
    n = 9
    bx = 2.0 * (n + 1)
    a = sk.gen_convdiff3d(n, bx, 1.0, 1.0)
    b = O.gen_convdiff3d(n, bx, 1.0, 1.0).csr()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


# ------------------------------------------------------------ incremental QR

def test_qr_matches_appended_columns(sk):  # test_incremental_qr.cpp:28-60
    rng = np.random.default_rng(1)
    M = rng.standard_normal((40, 12))
    qr = sk.IncrementalQR(40, 4)
    for j in range(12):
        col, rd = qr.append(M[:, j])
        assert col == j and not rd
    Q, R = qr.factors()
    assert np.linalg.norm(Q @ R - M) <= 1e-13 * np.linalg.norm(M)
    assert np.linalg.norm(Q.T @ Q - np.eye(12)) <= 1e-13
    b = rng.standard_normal(40)
    y, res = qr.solve(b)
    yr = np.linalg.lstsq(M, b, rcond=None)[0]
    assert np.linalg.norm(y - yr) <= 1e-12 * np.linalg.norm(yr)
    assert res == pytest.approx(np.linalg.norm(b - M @ yr), rel=1e-12)


def test_qr_graded_columns_stay_orthonormal(sk):  # test_incremental_qr.cpp:62-73
    rng = np.random.default_rng(2)
    M = rng.standard_normal((30, 10)) @ np.diag(10.0 ** -np.arange(10))
    qr = sk.IncrementalQR(30, 10)
    for j in range(10):
        qr.append(M[:, j])
    Q, _ = qr.factors()
    assert np.linalg.norm(Q.T @ Q - np.eye(10)) <= 1e-12


def test_qr_sentinel_exclude_and_relative_rank(sk):  # test_incremental_qr.cpp:75-123
    rng = np.random.default_rng(3)
    a, b = rng.standard_normal(20), rng.standard_normal(20)
    qr = sk.IncrementalQR(20, 3)
    qr.append(a)
    qr.append(b)
    col, rd = qr.append(2 * a - 3 * b)
    assert rd and col == 2
    with pytest.raises(sk.SdrError, match="column 2 is rank-deficient and unresolved"):
        qr.solve(rng.standard_normal(20))
    qr.exclude(2)
    y, _ = qr.solve(a)
    assert y[2] == 0.0 and y[0] == pytest.approx(1.0)
    small = sk.IncrementalQR(20, 2)
    small.append(1e-20 * a)
    col, rd = small.append(1e-20 * (a + 1e-3 * b))
    assert not rd  # the rank test is relative to the column norm
    with pytest.raises(ValueError, match="column length 19 does not match 20 rows"):
        qr.append(np.ones(19))
    with pytest.raises(ValueError):
        qr.exclude(7)


# ------------------------------------------------------------------ harmonic

def test_harmonic_matches_oracle_subspace(sk, O):  # test_recycle.cpp:87-129
    rng = np.random.default_rng(4)
    for p in (8, 30):
        SAW = rng.standard_normal((60, p))
        SW = rng.standard_normal((60, p))
        h = sk.harmonic_pairs(SAW, SW, 4)
        ho = O.harmonic(SAW, SW, 4)
        assert h["k_effective"] == ho["k_effective"] and h["rank"] == ho["rank"]
        A, B = sl.orth(h["coeffs"]), sl.orth(ho["coeffs"])
        assert np.linalg.norm(A - B @ (B.T @ A)) <= 1e-10
        assert np.allclose(np.sort(np.abs(h["mu"])), np.sort(np.abs(ho["mu"])), rtol=1e-10)


def test_harmonic_via_solver_qr_matches_oracle(sk, O):
    """The solver's route (QR factors of SAW; no SVD when R is well conditioned)
    extracts the same values and subspace as the reference's SVD route."""
    rng = np.random.default_rng(9)
    for p, scale in ((8, 1.0), (30, 1.0), (60, 1e-3)):
        SAW = rng.standard_normal((120, p)) * np.logspace(0, np.log10(scale), p)
        SW = rng.standard_normal((120, p))
        for k in (1, 4, min(20, p)):
            h = sk.harmonic_pairs(SAW, SW, k, via_qr=True)
            ho = O.harmonic(SAW, SW, k)
            assert h["k_effective"] == ho["k_effective"] and h["rank"] == ho["rank"] == p
            A, B = sl.orth(h["coeffs"]), sl.orth(ho["coeffs"])
            assert np.linalg.norm(A - B @ (B.T @ A)) <= 1e-9
            assert np.allclose(np.sort(np.abs(h["mu"])), np.sort(np.abs(ho["mu"])), rtol=1e-9)
    # numerically rank-deficient SAW: the QR route falls back to the truncated SVD
    U = rng.standard_normal((40, 5))
    SAW = np.column_stack([U, U[:, :2] @ rng.standard_normal((2, 3))])
    SW = rng.standard_normal((40, 8))
    h = sk.harmonic_pairs(SAW, SW, 3, via_qr=True)
    ho = O.harmonic(SAW, SW, 3)
    assert h["rank"] == ho["rank"] == 5 and h["k_effective"] == ho["k_effective"]


def test_harmonic_conjugate_pair_and_rank_limit(sk):  # test_recycle.cpp:131-185
    rng = np.random.default_rng(55)
    Q = np.linalg.qr(rng.standard_normal((4, 4)))[0]
    T0 = np.array([[3.0, 0, 0, 0], [0, 2.0, 1.0, 0], [0, -1.0, 2.0, 0], [0, 0, 0, 0.5]])
    U = np.linalg.qr(rng.standard_normal((20, 4)))[0]
    V = np.linalg.qr(rng.standard_normal((10, 4)))[0]
    h = sk.harmonic_pairs(U @ V.T, U @ (Q @ T0 @ Q.T) @ V.T, 2)
    assert h["k_effective"] == 3 and h["pair_extended"]
    assert abs(np.sum(h["mu"]) - 7.0) <= 1e-10 and abs(np.prod(h["mu"]) - 15.0) <= 1e-9
    lib_coords = V.T @ h["coeffs"]
    A, B = sl.orth(lib_coords), Q[:, :3]
    assert np.linalg.norm(A - B @ (B.T @ A)) <= 1e-10
    SAW = np.linalg.qr(rng.standard_normal((15, 2)))[0] @ np.linalg.qr(rng.standard_normal((6, 2)))[0].T
    h = sk.harmonic_pairs(SAW, rng.standard_normal((15, 6)), 5)
    assert h["rank"] == 2 and h["rank_limited"] and h["k_effective"] <= 2
    assert sk.harmonic_pairs(SAW, rng.standard_normal((15, 6)), 0)["k_effective"] == 0
    with pytest.raises(ValueError):
        sk.harmonic_pairs(SAW, SAW, -1)


# ----------------------------------------------------------------- partition

def test_partition_rows_zslabs(sk):
    rb, re = sk.partition_rows(512 ** 3, 8, 512 * 512)
    assert rb[0] == 0 and re[-1] == 512 ** 3 and np.all(rb[1:] == re[:-1])
    assert np.all((re - rb) == 64 * 512 * 512)
    rb, re = sk.partition_rows(10 * 16, 3, 16)
    assert (re - rb).tolist() == [48, 48, 64]
    with pytest.raises(ValueError):
        sk.partition_rows(100, 2, 7)


def test_partition_halo_plan_is_symmetric(sk):
    n2 = 16
    world = 4
    rb, re = sk.partition_rows(64 * n2, world, n2)
    mn = np.maximum(rb - n2, 0)
    mx = np.minimum(re - 1 + n2, 64 * n2 - 1)
    plans = [sk.partition_halo(r, rb, re, mn, mx) for r in range(world)]
    for p in range(world):
        for q in range(world):
            assert plans[p]["recv_cnt"][q] == plans[q]["send_cnt"][p]
            assert plans[p]["recv_lo"][q] == plans[q]["send_lo"][p]
        assert plans[p]["recv_cnt"].sum() == (rb[p] - mn[p]) + (mx[p] + 1 - re[p])
    assert plans[0]["recv_cnt"].tolist() == [0, n2, 0, 0]
    assert plans[1]["recv_lo"][0] == rb[1] - n2 and plans[1]["recv_lo"][2] == re[1]


def test_campaign_out_dir_resolution_and_solver_names(monkeypatch):
    """campaign.cpp:185-193 (test_campaign.cpp output-directory case)."""
    from paper_2311_14206_b200 import campaign as cp
    monkeypatch.delenv("SKRYLOV_OUT_DIR", raising=False)
    assert cp.resolve_out_dir("explicit", "fallback") == "explicit"
    assert cp.resolve_out_dir("", "fallback") == "fallback"
    monkeypatch.setenv("SKRYLOV_OUT_DIR", "from-env")
    assert cp.resolve_out_dir("", "fallback") == "from-env"
    assert cp.resolve_out_dir("explicit", "fallback") == "explicit"
    assert [cp.known_solver(s) for s in ("gmres-sdr", "sgmres", "gmres", "cg")] == [True, True, True, False]
    assert cp.num(0.1) == "0.10000000000000001" and cp.num(float("nan")) == "nan"


@pytest.mark.parametrize("g,shift", [(2, 0.0), (5, 0.1), (103, 1e-4), (12, 0.5)])
def test_gen_neumann_matches_oracle(sk, O, g, shift):
    """problems.hpp:38-61 (mirrored neighbours, duplicates summed): CSR identical to the oracle's."""
    off, col, val = sk.gen_neumann(g, shift)
    oo, oc, ov = O.gen_neumann(g, shift).csr()
    assert np.array_equal(off, oo) and np.array_equal(col, oc) and np.array_equal(val, ov)
    # the unshifted operator's rows sum to zero (all-ones null space)
    off0, col0, val0 = sk.gen_neumann(g, 0.0)
    sums = np.add.reduceat(val0, off0[:-1])
    assert np.all(sums == 0.0)
    with pytest.raises(ValueError):
        sk.gen_neumann(1, 0.0)


def test_config_any_window(sk):
    """Any t >= 1 validates, as in the reference (solver.hpp:61-70): windows
    past the fused kernels' 33 run the unfused wide path."""
    sk.SolverConfig(m=100, t=33, k=20, s=240, tol=1e-8).validate()
    sk.SolverConfig(m=100, t=100, k=20, s=240, tol=1e-8).validate()
    with pytest.raises(ValueError):
        sk.SolverConfig(m=100, t=0, k=20, s=240, tol=1e-8).validate()
