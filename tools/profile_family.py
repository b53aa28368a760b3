"""Where the time goes in the acceptance grid family (50 rhs, 103^2 Neumann
grid, m=100 t=2 k=20 s=1200 tol=1e-6): per-phase host wall time summed over
the sequence, per-kernel device time. Usage: python tools/profile_family.py [--count 50] [--s 1200]"""
import argparse
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402
from oracle import pyoracle as O  # noqa: E402  (test-side generator of the acceptance operator)

ap = argparse.ArgumentParser()
ap.add_argument("--count", type=int, default=50)
ap.add_argument("--s", type=int, default=1200)
ap.add_argument("--timing", action="store_true")
args = ap.parse_args()
ctx = sk.default_context()
M = O.gen_neumann(103, 1e-4)
off, col, val = M.csr()
G = sk.SparseMatrix(M.rows, M.cols, off, col, val)
rhs = [sk.gaussian_vector(M.rows, 2026 + i) for i in range(args.count)]
cfg = sk.SolverConfig(m=100, t=2, k=20, s=args.s, tol=1e-6, max_restarts=10)
S = sk.SketchOperator.subsampled_dct(M.rows, args.s, cfg.sketch_seed)
run = lambda: sk.solve_sequence([sk.ProblemInstance(G, x, target_tol=1e-6) for x in rhs], cfg, sketch=S,
                                shared_matrix=True)
run()
ctx.synchronize()
if args.timing:
    ctx.set_timing(True)
    ctx.timing_reset()
t = time.perf_counter()
seq = run()
ctx.synchronize()
wall = time.perf_counter() - t
ph = collections.Counter()
for r in seq.reports:
    for k, v in r.phases.items():
        ph[k] += v
out = {"wall_s": wall, "steps": sum(r.iterations for r in seq.reports),
       "iterations": [r.iterations for r in seq.reports][:10],
       "cycles": [r.cycles for r in seq.reports][:10],
       "phases_ms": {k: round(v, 2) for k, v in sorted(ph.items(), key=lambda kv: -kv[1])}}
if args.timing:
    ks = ["spmv_arnoldi", "update_sketch", "sketch_fold", "update_sketch_flush", "recycle_gemm", "col_norms",
          "residual", "spmv", "copy_norm", "axpy", "sketch", "sketch_tiles", "update", "tallskinny"]
    out["kernels"] = {k: ctx.timing(k) for k in ks if ctx.timing(k)[0]}
print(json.dumps(out))
