import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2311_14206_b200 as sk
from oracle import pyoracle as O
n, count = 128, 3
N = n*n
b0 = sk.gaussian_vector(N, 0x3000)
mats, omats, rhs = [], [], []
for i in range(count):
    d_rel = 1e-3 * (2.0 * sk.uniform_stream(0x3100 + i, N) - 1.0)
    off, col, val = sk.gen_convdiff2d(n, 100.0 + 2 * i, 100.0 - 2 * i, 0.01 * i, d_rel)
    mats.append(sk.SparseMatrix(N, N, off, col, val))
    omats.append(O.SparseMatrix.from_csr(N, N, off, col, val))
    rhs.append(b0 + 0.05 * sk.gaussian_vector(N, 0x3000 + i) if i else b0)
kw = dict(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact")
res = sk.solve_sequence([sk.ProblemInstance(A, b, target_tol=1e-8) for A, b in zip(mats, rhs)], sk.SolverConfig(**kw))
xs, reps = O.solve_sequence(omats, rhs, O.SolverConfig(**kw), tols=[1e-8] * count)
for i,(g,o) in enumerate(zip(res.reports, reps)):
    print("sys", i, g.status, o.status, g.iterations, o.iterations, g.counters, o.counters)
    print("  g defl", [c['deflation_rank'] for c in g.cycle_stats])
    print("  o defl", [c['deflation_rank'] for c in o.cycle_stats])
    print("  g notes", g.notes)
    print("  o notes", o.notes)
