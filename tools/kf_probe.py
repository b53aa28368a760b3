"""KF (fused step) probe: in-solve CUDA-event durations of the step kernels on
a 3-D convection-diffusion operator with the sparse-sign sketch (one cycle).
Usage: [SDR_KF_MODE=..] [SDR_FUSE_STEP=0] python tools/kf_probe.py [--n 512] [--m 20]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--m", type=int, default=20)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
A = sk.SparseMatrix.convdiff3d_device(args.n, 200.0, 100.0, 50.0)
N = A.rows
b = sk.gaussian_vector(N, 3)
S = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8)
cfg = sk.SolverConfig(m=args.m, k=10, t=2, s=120, tol=1e-30, max_restarts=1)
ctx = A.ctx
sk.solve(A, b, cfg, sketch=S)
ctx.set_timing(True)
for _ in range(args.reps):
    ctx.timing_reset()
    sk.solve(A, b, cfg, sketch=S)
    ctx.synchronize()
    out = []
    for k in ("fused_step", "fused_fold", "spmv_arnoldi", "update_sketch", "sketch_fold"):
        n, ms = ctx.timing(k)
        if n:
            out.append(f"{k} {n}x {1e3 * ms / n:.1f}us")
    print(f"mode={os.environ.get('SDR_KF_MODE', '0')} fuse={os.environ.get('SDR_FUSE_STEP', '1')}: " + ", ".join(out),
          flush=True)
