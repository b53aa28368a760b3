"""C5 step kernels in isolation: the 512^3 operator, sparse sign ζ=8, and a
few truncated-Arnoldi steps through sdr_krylov_run with per-launch CUDA-event
timing. Short enough to run under ncu (-k regex:<kernel> -c 1).
Usage: python tools/profile_c5_step.py [steps] [n]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
ctx = sk.default_context()
A = sk.SparseMatrix.convdiff3d_device(n, 200.0, 100.0, 50.0, ctx=ctx)
N = A.rows
S = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8, ctx=ctx)
r0 = sk.gaussian_vector(N, 3)
m, t, s = steps, 2, 120
V = np.zeros((m + 1) * N)
H = np.zeros((m + 1) * m)
SV = np.zeros(s * (m + 1))
SAV = np.zeros(s * m)
j, br, rn = C.c_int64(), C.c_int(), C.c_double()
cnt = np.zeros(3, dtype=np.int64)
p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
for rep in range(2):
    ctx.set_timing(rep == 1)
    ctx.timing_reset()
    sk._check(sk._lib.sdr_krylov_run(ctx._h, A._h, S._h, p(r0), t, m, m, 1e-14, p(V), p(H), p(SV), p(SAV), C.byref(j),
                                     C.byref(br), C.byref(rn), p(cnt)))
    ctx.synchronize()
for name in ("spmv_arnoldi", "update", "update_sketch", "sketch", "sketch_fold", "fold_partials", "copy_norm"):
    c, ms = ctx.timing(name)
    if c:
        print(f"{name:14s} n={c:3d} avg {1e3 * ms / c:9.1f} us")
print("H diag", H.reshape(m, m + 1).T[0, 0], "SV norm", np.linalg.norm(SV))
