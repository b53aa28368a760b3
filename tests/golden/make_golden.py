"""Generates tests/golden/*.json from the CPU oracle (oracle/, the C++
restatement of the reference). The GPU tests compare the sm_100a path with
these fixtures at BASELINE sizes where rerunning the oracle would take
minutes. Run: python tests/golden/make_golden.py [c1 c2 c3 small]"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np  # noqa: E402

from oracle import pyoracle as O  # noqa: E402


def summary(x, rep, extra=None):
    d = dict(status=rep.status, iterations=rep.iterations, cycles=rep.cycles, rhs_norm=rep.rhs_norm,
             final_relative_residual=rep.final_relative_residual, counters=rep.counters,
             sketched_residuals=rep.sketched_residuals, true_residuals=rep.true_residuals,
             cycle_stats=rep.cycle_stats, notes=rep.notes, seconds=rep.seconds,
             x_head=x[:16].tolist(), x_norm=float(np.linalg.norm(x)))
    d.update(extra or {})
    return d


def c1():
    """BASELINE C1: A = -gen_convdiff(100, -50), b = N(0,1) seed 0 normalised, m=50 k=10 t=2 s=120, tol 1e-8."""
    off, col, val = O.gen_convdiff(100, -50.0).csr()
    A = O.SparseMatrix.from_csr(10000, 10000, off, col, -val)
    b = O.gaussian_vector(10000, 0)
    b /= np.linalg.norm(b)
    out = {}
    for name, S in (("srdct", None), ("sparse_sign", O.SketchOperator.sparse_sign(10000, 120, 0x5EED, 8))):
        cfg = O.SolverConfig(m=50, k=10, t=2, s=120, tol=1e-8, max_restarts=40)
        x, rep = O.solve(A, b, cfg, sketch=S)
        out[name] = summary(x, rep, dict(config=dict(m=50, k=10, t=2, s=120, tol=1e-8, max_restarts=40)))
    return out


def c2():
    """BASELINE C2: 3D 128^3, beta=(100,50,25), b = gaussian_vector(N, 1), m=100 k=20 t=2 s=240 tol 1e-8."""
    n = 128
    A = O.gen_convdiff3d(n, 100.0, 50.0, 25.0)
    b = O.gaussian_vector(n ** 3, 1)
    cfg = O.SolverConfig(m=100, k=20, t=2, s=240, tol=1e-8)
    t0 = time.time()
    x, rep = O.solve(A, b, cfg)
    return summary(x, rep, dict(config=dict(n=n, m=100, k=20, t=2, s=240, tol=1e-8), wall_s=time.time() - t0))


def c3_small():
    """C3-shaped sequence at a CPU-friendly size (64^2 grid, 5 systems)."""
    n, count = 64, 5
    rng = O
    b0 = O.gaussian_vector(n * n, 0x3000)
    mats, rhss = [], []
    for i in range(count):
        rel = 1e-3 * (2.0 * O.uniform_stream(0x3100 + i, n * n) - 1.0)
        mats.append(O.gen_convdiff2d(n, 100.0 + 2 * i, 100.0 - 2 * i, 0.01 * i, rel))
        rhss.append(b0 + 0.05 * O.gaussian_vector(n * n, 0x3000 + i) if i else b0.copy())
    cfg = O.SolverConfig(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact", max_restarts=20)
    xs, reps = O.solve_sequence(mats, rhss, cfg)
    return [summary(x, r) for x, r in zip(xs, reps)]


def c3_first():
    """BASELINE C3 at full size, its first system alone (N = 1024^2, same
    construction and seeds as tools/bench_sequence.py; ~3 min on one core)."""
    n = 1024
    b0 = O.gaussian_vector(n * n, 0x3000)
    rel = 1e-3 * (2.0 * O.uniform_stream(0x3100, n * n) - 1.0)
    A = O.gen_convdiff2d(n, 100.0, 100.0, 0.0, rel)
    cfg = O.SolverConfig(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact")
    x, rep = O.solve(A, b0, cfg)
    return summary(x, rep, dict(config=dict(n=n, m=50, k=20, t=2, s=140, tol=1e-8, variant="exact")))


def c4_complex():
    """BASELINE C4 with complex GMRES-SDR (oracle/skrylov_oracle_complex.hpp;
    parity unpinned against the reference, which has no complex solver): the
    full 32^3 x 64 lattice, m0 = -0.8, theta seed 2, b = gaussian_vector(2N, 4)
    as (re, im) pairs, m=80 k=20 t=3 s=200 tol=1e-8, SRDCT(N, 200, 0x5eed) on
    Re / Im; then the 10-system sequence m0 += 0.01 with the recycle space
    carried and refreshed exactly (SAU = S A_i U). Also the realified solve's
    counts on a reduced lattice for comparison (tools/c4_problem.py)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from tools.c4_problem import c4_complex_csr, c4_csr
    dims = (32, 32, 32, 64)
    N = int(np.prod(dims))
    g = O.gaussian_vector(2 * N, 4)
    b = g[0::2] + 1j * g[1::2]
    S = O.SketchOperator.subsampled_dct(N, 200, 0x5EED)
    kw = dict(m=80, k=20, t=3, s=200, tol=1e-8, max_restarts=40)
    out = {"config": dict(dims=list(dims), m0=-0.8, **kw), "sequence": []}
    space = O.ZRecycleSpace()
    for i in range(10):
        off, col, val = c4_complex_csr(dims, m0=-0.8 + 0.01 * i, seed=2, uniform=O.uniform_stream)
        A = O.ZSparseMatrix(N, off, col, val)
        del off, col, val
        ref = space.refresh(A, S) if i > 0 and space.dim > 0 else dict(matvecs=0, inner_products=0, sketch_applies=0)
        x, rep = O.zsolve(A, b, O.SolverConfig(**kw), S, space=space)
        d = dict(status=rep.status, iterations=rep.iterations, cycles=rep.cycles,
                 final_relative_residual=rep.final_relative_residual, counters=rep.counters, refresh=ref,
                 true_residuals=rep.true_residuals, x_norm=float(np.linalg.norm(x)))
        if i == 0:
            out["single"] = d
        out["sequence"].append(d)
        print(f"  c4 system {i}: {rep.status} {rep.iterations} it", flush=True)
    small = {}
    for sd in [(4, 4, 4, 8), (8, 8, 8, 16), (16, 16, 16, 32)]:
        n = int(np.prod(sd))
        oc, cc, vc = c4_complex_csr(sd, -0.8, 2, O.uniform_stream)
        gz = O.gaussian_vector(2 * n, 4)
        xz, rz = O.zsolve(O.ZSparseMatrix(n, oc, cc, vc), gz[0::2] + 1j * gz[1::2], O.SolverConfig(**kw),
                          O.SketchOperator.subsampled_dct(n, 200, 0x5EED))
        orr, cr, vr = c4_csr(sd, -0.8, 2, O.uniform_stream)
        xr, rr = O.solve(O.SparseMatrix.from_csr(2 * n, 2 * n, orr, cr, vr), gz, O.SolverConfig(**kw),
                         sketch=O.SketchOperator.subsampled_dct(2 * n, 200, 0x5EED))
        small["x".join(map(str, sd))] = dict(complex=dict(status=rz.status, iterations=rz.iterations),
                                             realified=dict(status=rr.status, iterations=rr.iterations))
    out["complex_vs_realified"] = small
    return out


def main(which):
    jobs = {"c1": c1, "c2": c2, "c3_small": c3_small, "c3_first": c3_first, "c4_complex": c4_complex}
    for name in which:
        t0 = time.time()
        data = jobs[name]()
        path = os.path.join(HERE, f"{name}_oracle.json")
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1)
        print(f"{name}: wrote {path} in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c3_small", "c2", "c3_first"])
