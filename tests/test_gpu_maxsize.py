"""Maximum-size checks at BASELINE C5 (512^3 = 134 M rows, 938 M stored
entries, built directly in HBM): the device SpMV agrees, on slabs at both
ends and in the middle of the grid, with the host CSR generator applied on
the CPU in CSR order; the sparse-sign sketch at full length is linear and
deterministic; the SRDCT at N = 2^27 matches its closed form on a sparse
input (size-independent properties)."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def test_c5_spmv_slabs_match_host_csr(sk):
    import torch
    n = 512
    beta = (200.0, 100.0, 50.0)
    A = sk.SparseMatrix.convdiff3d_device(n, *beta)
    N = n ** 3
    assert A.rows == N and A.storage["format"] == "dia"
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
    y = A.apply(x)
    plane = n * n
    for z0, z1 in ((0, 2), (255, 257), (510, 512)):
        off, col, val = sk.gen_convdiff3d(n, *beta, z_begin=z0, z_end=z1)
        lo, hi = max(0, z0 - 1) * plane, min(n, z1 + 1) * plane  # the columns the slab rows reach
        xs = x[lo:hi].cpu().numpy()
        M = sp.csr_matrix((val, col - lo, off), shape=((z1 - z0) * plane, hi - lo))
        ref = M @ xs
        got = y[z0 * plane:z1 * plane].cpu().numpy()
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_c5_sparse_sign_linear_and_deterministic(sk):
    import torch
    N = 512 ** 3
    S = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8)
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
    sa, sb = S.apply(a), S.apply(b)
    sab = S.apply(2.0 * a - 3.0 * b)
    assert np.linalg.norm(sab - (2.0 * sa - 3.0 * sb)) <= 1e-13 * np.linalg.norm(sab)
    assert np.array_equal(S.apply(a), sa)
    # ||S a||^2 / ||a||^2 near 1 (unbiased embedding, 120 rows)
    ratio = np.dot(sa, sa) / float(torch.dot(a, a))
    assert 0.6 < ratio < 1.6


def test_srdct_2p27_known_answer_on_sparse_input(sk):
    """SRDCT at N = 2^27 (the four-step tile path): S x for a vector with a
    few nonzeros against the closed form sqrt(n/s) alpha_k sign_j cos(pi k (2j+1) / 2N),
    phases reduced exactly in integers."""
    import torch
    N, s = 1 << 27, 120
    S = sk.SketchOperator.subsampled_dct(N, s, 0x5EED)
    rows = S.rows().astype(np.int64)
    signs = S.signs()
    rng = np.random.default_rng(11)
    js = np.sort(rng.choice(N, 5, replace=False))
    cs = rng.standard_normal(5)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    x[torch.from_numpy(js).cuda()] = torch.from_numpy(cs).cuda()
    got = S.apply(x)
    ref = np.zeros(s)
    for j, c in zip(js, cs):
        ph = (rows * (2 * int(j) + 1)) % (4 * N)  # exact phase, units of pi / 2N
        ref += c * signs[j] * np.cos(np.pi * ph / (2.0 * N))
    alpha = np.where(rows == 0, np.sqrt(1.0 / N), np.sqrt(2.0 / N))
    ref *= alpha * np.sqrt(N / s)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
