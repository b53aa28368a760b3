"""Short C2 driver for ncu captures: one warm-up solve, then `--steps`
Arnoldi steps through sdr_krylov_run (the per-step kernels K1/K2/K3)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--solve", action="store_true", help="run a full warm solve first")
args = ap.parse_args()

n = 128
A = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0)
N = A.rows
b = sk.gaussian_vector(N, 1)
S = sk.SketchOperator.subsampled_dct(N, 240, 0x5EED)
if args.solve:
    r = sk.solve(A, b, sk.SolverConfig(m=100, k=20, t=2, s=240, tol=1e-8), sketch=S)
    print("solve", r.report.status, r.report.iterations, {k: round(v, 2) for k, v in r.report.phases.items()})
m = 100
j, br, rn = C.c_int64(), C.c_int(), C.c_double()
sk._check(sk._lib.sdr_krylov_run(A.ctx._h, A._h, S._h, b.ctypes.data_as(C.c_void_p), 2, m, args.steps, 1e-14,
                                 None, None, None, None, C.byref(j), C.byref(br), C.byref(rn), None))
print("krylov steps", j.value)
