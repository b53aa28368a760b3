"""Acceptance criteria 2, 5 and 10 (proj/tests/acceptance.cpp:85-131,
194-234, 358-401) on the device Arnoldi path: the basis, sketched blocks
and harmonic values come from the B200 kernels (sdr_krylov_run /
sdr_harmonic); the dense checks (distortion, least squares, harmonic Ritz
values) are computed here in numpy as the reference's test oracle does."""
import numpy as np
import pytest
import scipy.linalg as sl

from tests.test_gpu_parity import krylov

pytestmark = pytest.mark.gpu


def random_shifted(O, n, seed, shift):
    """acceptance.cpp:43-51: gaussian entries / sqrt(n), column-major fill, + shift I."""
    A = O.gaussian_vector(n * n, seed).reshape(n, n).T / np.sqrt(n)
    return A + shift * np.eye(n)


def orth(X):
    Q, R, _ = sl.qr(X, mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    r = int(np.sum(d > d[0] * max(X.shape) * np.finfo(float).eps)) if d.size else 0
    return Q[:, :r]


def distortion(Sd, span):
    s = np.linalg.svd(Sd @ orth(span), compute_uv=False)
    return float(np.max(np.abs(s * s - 1.0)))


def test_criterion2_residual_chain(sk, O):
    slack = 1.0 + 1e-12
    for i in range(20):
        m = 3 + i % 10
        n = max(80 + (i * 7) % 21, 8 * m + 1)
        A = random_shifted(O, n, 300 + i, 2.0)
        b = O.gaussian_vector(n, 400 + i)
        S = sk.SketchOperator.subsampled_dct(n, 8 * m, 500 + i)
        g = krylov(sk, sk.SparseMatrix.from_dense(A), S, b, 2, m)
        assert g["j"] == m and not g["breakdown"]
        AV = A @ g["V"][:, :m]
        Sd = S.dense()
        sr0 = Sd @ b
        r_true = b - AV @ np.linalg.lstsq(AV, b, rcond=None)[0]
        r_sk = b - AV @ np.linalg.lstsq(Sd @ AV, sr0, rcond=None)[0]
        eps = distortion(Sd, np.column_stack([b, AV]))
        assert eps < 1.0
        root = np.sqrt(1.0 - eps)
        q = [np.linalg.norm(r_true), np.linalg.norm(r_sk), np.linalg.norm(Sd @ r_sk) / root,
             np.linalg.norm(Sd @ r_true) / root, np.sqrt((1 + eps) / (1 - eps)) * np.linalg.norm(r_true)]
        assert all(q[k] <= q[k + 1] * slack for k in range(4)), (i, q)


def test_criterion5_harmonic_values_match_dense_ritz(sk, O):
    worst = 0.0
    for i in range(10):
        n, m, k = 60 + 4 * i, 15, 2 + i % 9
        A = random_shifted(O, n, 900 + i, 2.0)
        b = O.gaussian_vector(n, 1000 + i)
        S = sk.SketchOperator.identity(n)
        g = krylov(sk, sk.SparseMatrix.from_dense(A), S, b, m, m)  # full window
        assert g["j"] == m and not g["breakdown"]
        hp = sk.harmonic_pairs(g["SAV"][:, :m], g["SV"][:, :m], k)
        assert hp["k_effective"] >= 1
        lib = list(1.0 / hp["mu"])
        # dense harmonic Ritz values over the m-step Krylov space
        W = orth(g["V"][:, :m])  # the m-step Krylov space
        AW = A @ W
        theta = sl.eigvals(AW.T @ AW, AW.T @ W)
        ref = sorted(theta, key=lambda z: (abs(z), -z.real))[: len(lib)]
        # pair values by nearest match (the two members of a conjugate pair
        # may differ in the last bits of their real parts, which breaks a
        # (real, imag) sort)
        for a in lib:
            d = [abs(a - r) / max(1.0, abs(r)) for r in ref]
            worst = max(worst, min(d))
            ref.pop(int(np.argmin(d)))
    assert worst <= 1e-8, worst


def test_criterion10_angle_bound(sk, O):
    for i in range(10):
        n, m = 64 + 4 * i, 10
        A = random_shifted(O, n, 4000 + i, 2.0)
        b = O.gaussian_vector(n, 4100 + i)
        S = sk.SketchOperator.subsampled_dct(n, 56, 4200 + i)
        Sd = S.dense()
        g = krylov(sk, sk.SparseMatrix.from_dense(A), S, b, 2, m)
        assert g["j"] == m and not g["breakdown"]
        sr0 = Sd @ b
        nb = np.linalg.norm(b)
        for j in range(1, m + 1):
            AVj = A @ g["V"][:, :j]
            y = np.linalg.lstsq(Sd @ AVj, sr0, rcond=None)[0]
            res = np.linalg.norm(b - AVj @ y)
            Q = orth(AVj)
            cosa = min(1.0, np.linalg.norm(Q.T @ b) / nb)
            sina = np.linalg.norm(b - Q @ (Q.T @ b)) / nb
            eps = distortion(Sd, np.column_stack([b, AVj]))
            assert eps < 1.0
            bound = nb * np.sqrt((sina ** 2 + 2.0 * eps * (1.0 + cosa)) / (1.0 - eps ** 2))
            assert res <= bound * (1.0 + 1e-10), (i, j, res, bound)
