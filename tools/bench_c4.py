"""BASELINE C4 on one GPU through the real-equivalent system (tools/c4_problem.py):
32^3 x 64 sites, m0 = -0.8, theta seed 2, b = gaussian_vector(2N, 4) interleaved,
m=80 k=20 t=3 s=200 tol=1e-8; then the 10-system sequence m0 += 0.01 (same
phases and rhs; the recycle space carried, variant exact).
Usage: python tools/bench_c4.py [--dims 32 32 32 64] [--sequence 10]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402
from tools.c4_problem import c4_csr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[32, 32, 32, 64])
ap.add_argument("--sequence", type=int, default=10)
ap.add_argument("--steps", type=int, default=1)
args = ap.parse_args()
ctx = sk.default_context()
t0 = time.time()
mats = []
for i in range(max(1, args.sequence)):
    off, col, val = c4_csr(tuple(args.dims), m0=-0.8 + 0.01 * i, seed=2, uniform=sk.uniform_stream)
    n2 = len(off) - 1
    mats.append(sk.SparseMatrix(n2, n2, off, col, val, ctx=ctx))
    del off, col, val
setup_s = time.time() - t0
n2 = mats[0].rows
import torch  # noqa: E402
b = torch.from_numpy(sk.gaussian_vector(n2, 4)).cuda()  # resident in HBM, like bench.py's value
cfg = sk.SolverConfig(m=80, k=20, t=3, s=200, tol=1e-8, variant="exact")
S = sk.SketchOperator.subsampled_dct(n2, 200, cfg.sketch_seed, ctx=ctx)
sk.solve(mats[0], b, cfg, sketch=S)  # warm-up
ctx.synchronize()
t1 = time.perf_counter()
single = [sk.solve(mats[0], b, cfg, sketch=S) for _ in range(args.steps)]
ctx.synchronize()
t_single = (time.perf_counter() - t1) / args.steps
r = single[-1].report
seq = None
if args.sequence > 1:
    t2 = time.perf_counter()
    out = sk.solve_sequence([sk.ProblemInstance(A, b) for A in mats], cfg, sketch=S)
    ctx.synchronize()
    t_seq = time.perf_counter() - t2
    seq = {"iterations": [x.iterations for x in out.reports], "status": [x.status for x in out.reports],
           "wall_s": round(t_seq, 4), "steps_per_s": sum(x.iterations for x in out.reports) / t_seq}
print(json.dumps({
    "metric": "gmres_sdr_arnoldi_steps_per_s", "value": r.iterations / t_single, "unit": "steps/s", "n_gpus": 1,
    "ms_per_step": 1e3 * t_single, "dtype": "f64 (real-equivalent of complex fp64)", "data": "synthetic (C4 construction, seeded)",
    "config": {"workload": "c4", "sites": n2 // 2, "N_real": n2, "nnz_real": mats[0].nnz, "storage": mats[0].storage,
               "m": 80, "k": 20, "t": 3, "s": 200, "tol": 1e-8},
    "solve": {"status": r.status, "iterations": r.iterations, "cycles": r.cycles,
              "final_relative_residual": r.final_relative_residual},
    "sequence": seq, "setup_s": round(setup_s, 1)}), flush=True)
