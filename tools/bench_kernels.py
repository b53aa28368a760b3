"""Per-kernel CUDA-event timings of the Arnoldi step at C2 (sdr_krylov_run with
context timing on). Usage: python tools/bench_kernels.py [--steps 60] [--n 128]"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--sketch", default="srdct")
ap.add_argument("--s", type=int, default=240)
args = ap.parse_args()

ctx = sk.default_context()
A = sk.SparseMatrix.convdiff3d_device(args.n, 100.0, 50.0, 25.0)
N = A.rows
b = sk.gaussian_vector(N, 1)
S = (sk.SketchOperator.subsampled_dct(N, args.s, 0x5EED) if args.sketch == "srdct"
     else sk.SketchOperator.sparse_sign(N, args.s, 0x5EED, 8))


def run(steps):
    j, br, rn = C.c_int64(), C.c_int(), C.c_double()
    sk._check(sk._lib.sdr_krylov_run(ctx._h, A._h, S._h, b.ctypes.data_as(C.c_void_p), 2, 100, steps, 1e-14,
                                     None, None, None, None, C.byref(j), C.byref(br), C.byref(rn), None))
    return j.value


run(5)
ctx.set_timing(True)
ctx.timing_reset()
t0 = time.perf_counter()
run(args.steps)
wall = time.perf_counter() - t0
out = {"N": N, "nnz": A.nnz, "steps": args.steps, "wall_ms_per_step": 1e3 * wall / args.steps,
       "K1_PIPE": os.environ.get("SDR_K1_PIPE", "0")}
for k in ("spmv_arnoldi", "update", "sketch", "update_sketch", "copy_norm"):
    n, ms = ctx.timing(k)
    if n:
        out[k] = round(1e3 * ms / n, 2)
ctx.set_timing(False)
print(json.dumps(out))
