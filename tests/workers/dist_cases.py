"""Problems of the world-size-2 product-path test: each rank builds its z-slab
(or row block) with global column indices; world = 1 builds the whole
operator for the reference solve."""
import numpy as np

CASES = {
    # 32^3 convection-diffusion, sparse sign (C5's sketch): non-deferred pipeline
    "conv_sparse": dict(kind="conv3d", n=32, sketch="sparse_sign", m=30, k=8, t=2, s=120, tol=1e-8),
    # 32^3 with SRDCT (C2's sketch): the deferred pipeline, fused update + SRDCT, split K1
    "conv_srdct": dict(kind="conv3d", n=32, sketch="srdct", m=40, k=10, t=2, s=120, tol=1e-8),
    # 33^3 on two slabs of 16 and 17 planes (an odd row count on one rank):
    # the ranks must agree on one step pipeline although their slabs differ
    "conv_srdct_uneven": dict(kind="conv3d", n=33, sketch="srdct", m=40, k=10, t=2, s=120, tol=1e-8),
    # a CSR operator whose interior rows reach into the neighbour's rows
    # (non-uniform stencil reach: the K1 interior / boundary split must use
    # the per-row reach, not the halo width)
    "csr_reach": dict(kind="csr_reach", n=24, sketch="srdct", m=30, k=6, t=3, s=120, tol=1e-8),
    # the same with sparse sign: the non-deferred step's interior / boundary K1 split
    "csr_reach_sparse": dict(kind="csr_reach", n=24, sketch="sparse_sign", m=30, k=6, t=2, s=120, tol=1e-8),
}


def _csr_reach(sk, n):
    """Convection-diffusion on n^3 plus long-range couplings from a band of
    rows in the middle of each half: row r reads row r + N/2 (first half) or
    r - N/2 (second half), so at two ranks those interior rows depend on the
    neighbour's block while the rows around them do not."""
    off, col, val = sk.gen_convdiff3d(n, 100.0, 50.0, 25.0)
    N = n ** 3
    rows = np.repeat(np.arange(N), np.diff(off))
    h = N // 2
    extra_r = np.array([r for r in range(N) if h // 4 <= r % h < h // 4 + 512 and r % 7 == 0])
    extra_c = np.where(extra_r < h, extra_r + h, extra_r - h)
    r = np.concatenate([rows, extra_r])
    c = np.concatenate([col, extra_c])
    v = np.concatenate([val, np.full(len(extra_r), -1.0)])
    key = r * N + c
    order = np.argsort(key, kind="stable")
    r, c, v = r[order], c[order], v[order]
    uniq, first = np.unique(r * N + c, return_index=True)
    v = np.add.reduceat(v, first)
    r, c = r[first], c[first]
    offsets = np.zeros(N + 1, dtype=np.int64)
    np.add.at(offsets, r + 1, 1)
    return np.cumsum(offsets), c.astype(np.int64), v


def build(sk, p, ctx, rank, world):
    n = p["n"]
    N = n ** 3
    if p["kind"] == "conv3d":
        z0, z1 = n * rank // world, n * (rank + 1) // world
        A = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0, z_begin=z0, z_end=z1, ctx=ctx)
    else:
        off, col, val = _csr_reach(sk, n)
        n2 = n * n
        r0, r1 = (n * rank // world) * n2, (n * (rank + 1) // world) * n2
        if world == 1:
            A = sk.SparseMatrix(N, N, off, col, val, ctx)
        else:
            loff = off[r0:r1 + 1] - off[r0]
            A = sk.SparseMatrix(N, N, loff, col[off[r0]:off[r1]], val[off[r0]:off[r1]], ctx, row_begin=r0,
                                local_rows=r1 - r0)
    b = sk.gaussian_vector(N, 7)[A.row_begin:A.row_begin + A.local_rows].copy()
    S = (sk.SketchOperator.sparse_sign(N, p["s"], 0x5EED, 8, ctx=ctx) if p["sketch"] == "sparse_sign"
         else sk.SketchOperator.subsampled_dct(N, p["s"], 0x5EED, ctx=ctx))
    cfg = sk.SolverConfig(m=p["m"], k=p["k"], t=p["t"], s=p["s"], tol=p["tol"], max_restarts=40)
    return A, b, S, cfg
