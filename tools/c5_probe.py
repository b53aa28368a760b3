"""C5 convergence probe: 512^3 convdiff, sparse sign, m=50 k=10 t=2 s=120,
tol 1e-7, with max_restarts raised (argv[1], default 400). Prints per-cycle
residuals and the solve time on cuda:0."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

n = int(os.environ.get("C5_N", "512"))
restarts = int(sys.argv[1]) if len(sys.argv) > 1 else 400
ctx = sk.Context(0)
t0 = time.time()
A = sk.SparseMatrix.convdiff3d_device(n, 200.0, 100.0, 50.0, ctx=ctx)
N = A.rows
b = torch.from_numpy(sk.gaussian_vector(N, 3)).cuda()
S = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8, ctx=ctx)
print(f"setup {time.time() - t0:.1f} s, storage {A.storage}", flush=True)
cfg = sk.SolverConfig(m=50, k=10, t=2, s=120, tol=1e-7, max_restarts=restarts)
for rep_i in range(2):
    torch.cuda.synchronize()
    t1 = time.time()
    r = sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S)
    ctx.synchronize()
    dt = time.time() - t1
    rp = r.report
    print(f"solve {rep_i}: status={rp.status} iterations={rp.iterations} cycles={rp.cycles} "
          f"final_rel={rp.final_relative_residual:.3e} wall={dt:.2f} s steps/s={rp.iterations / dt:.1f}", flush=True)
    if rep_i == 0:
        for i, c in enumerate(rp.cycle_stats):
            if i < 5 or i % 10 == 0 or i == len(rp.cycle_stats) - 1:
                print(f"  cycle {i}: steps={c['steps']} exit_res={c['exit_residual'] / rp.rhs_norm:.3e} "
                      f"safety={c['safety_after']:.2f} defl={c['deflation_rank']}")
    print("phases", {k: round(v, 1) for k, v in rp.phases.items()}, flush=True)
