"""BASELINE C4 (complex fp64 4-D lattice operator) in its real-equivalent form.

The reference has no complex solver ("a compile-level variant, not
required"), so C4 is run here through the real path on the
realified system: complex x = xr + i xi is stored interleaved [xr_0, xi_0,
xr_1, xi_1, ...] and each complex entry a = ar + i ai becomes the 2x2 block
[[ar, -ai], [ai, ar]]. The solution is the same complex vector; the Krylov
method is real GMRES-SDR on the 2N-dimensional real system (not complex
GMRES-SDR — iteration counts differ from a complex solver).

Operator: L = 32^3 x 64 sites, lexicographic (x fastest),
diagonal 4 + m0, eight periodic neighbour couplings -0.5 e^{i theta}; theta =
2 pi Rng(seed).uniform() drawn site by site in the neighbour order
(+x, -x, +y, -y, +z, -z, +t, -t). b: complex N(0,1) = gaussian_vector(2N, seed
b_seed) interleaved (re, im)."""
import numpy as np


def c4_csr(dims=(32, 32, 32, 64), m0=-0.8, seed=2, uniform=None):
    """(offsets, columns, values) of the realified operator, int64 / float64."""
    X, Y, Z, T = dims
    N = X * Y * Z * T
    p = np.arange(N, dtype=np.int64)
    x, y, z, t = p % X, (p // X) % Y, (p // (X * Y)) % Z, p // (X * Y * Z)
    strides = (1, X, X * Y, X * Y * Z)
    coords = (x, y, z, t)
    sizes = (X, Y, Z, T)
    nbr = []
    for d in range(4):
        for sgn in (1, -1):
            c = (coords[d] + sgn) % sizes[d]
            nbr.append(p + (c - coords[d]) * strides[d])
    nbr = np.stack(nbr, axis=1)  # N x 8
    u = uniform(seed, 8 * N).reshape(N, 8)
    theta = 2.0 * np.pi * u
    cr, ci = -0.5 * np.cos(theta), -0.5 * np.sin(theta)
    # complex entries per site: diagonal first, then the 8 neighbours; sorted by column per row
    ccols = np.concatenate([p[:, None], nbr], axis=1)                   # N x 9
    car = np.concatenate([np.full((N, 1), 4.0 + m0), cr], axis=1)      # N x 9
    cai = np.concatenate([np.zeros((N, 1)), ci], axis=1)
    order = np.argsort(ccols, axis=1, kind="stable")
    ccols = np.take_along_axis(ccols, order, axis=1)
    car = np.take_along_axis(car, order, axis=1)
    cai = np.take_along_axis(cai, order, axis=1)
    # realified rows: 2p (re) -> cols 2q (ar), 2q+1 (-ai); 2p+1 (im) -> 2q (ai), 2q+1 (ar)
    cols_re = np.stack([2 * ccols, 2 * ccols + 1], axis=2).reshape(N, 18)
    vals_re = np.stack([car, -cai], axis=2).reshape(N, 18)
    vals_im = np.stack([cai, car], axis=2).reshape(N, 18)
    cols = np.stack([cols_re, cols_re], axis=1).reshape(2 * N, 18)
    vals = np.stack([vals_re, vals_im], axis=1).reshape(2 * N, 18)
    # the diagonal block has ai = 0: drop its exact zeros like from_triplets (sparse.hpp:66)
    keep = vals != 0.0
    counts = keep.sum(axis=1)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return offsets, cols[keep].astype(np.int64), vals[keep]


def c4_complex_csr(dims=(32, 32, 32, 64), m0=-0.8, seed=2, uniform=None):
    """(offsets, columns, values) of the complex operator itself (complex128
    values, columns sorted per row): the input of complex GMRES-SDR
    (sdr_csr_create_complex / SparseMatrix.from_complex)."""
    X, Y, Z, T = dims
    N = X * Y * Z * T
    p = np.arange(N, dtype=np.int64)
    x, y, z, t = p % X, (p // X) % Y, (p // (X * Y)) % Z, p // (X * Y * Z)
    strides = (1, X, X * Y, X * Y * Z)
    coords = (x, y, z, t)
    sizes = (X, Y, Z, T)
    nbr = []
    for d in range(4):
        for sgn in (1, -1):
            c = (coords[d] + sgn) % sizes[d]
            nbr.append(p + (c - coords[d]) * strides[d])
    nbr = np.stack(nbr, axis=1)
    theta = 2.0 * np.pi * uniform(seed, 8 * N).reshape(N, 8)
    cv = -0.5 * np.exp(1j * theta)
    ccols = np.concatenate([p[:, None], nbr], axis=1)
    cvals = np.concatenate([np.full((N, 1), 4.0 + m0, dtype=np.complex128), cv], axis=1)
    order = np.argsort(ccols, axis=1, kind="stable")
    ccols = np.take_along_axis(ccols, order, axis=1)
    cvals = np.take_along_axis(cvals, order, axis=1)
    offsets = np.arange(0, 9 * N + 1, 9, dtype=np.int64)
    return offsets, ccols.reshape(-1), cvals.reshape(-1)
