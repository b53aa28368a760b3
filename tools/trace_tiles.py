"""Per-CTA phase timeline of the last SRDCT tile-kernel launch (SDR_TRACE=1).
Usage: SDR_TRACE=1 python tools/trace_tiles.py [--steps 4]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--c3", action="store_true", help="C3's 1024^2 2-D operator, s = 140")
args = ap.parse_args()
assert os.environ.get("SDR_TRACE") == "1"
ctx = sk.default_context()
if args.c3:
    off, col, val = sk.gen_convdiff2d(1024, 100.0, 100.0)
    A = sk.SparseMatrix(1 << 20, 1 << 20, off, col, val, ctx=ctx)
    S = sk.SketchOperator.subsampled_dct(A.rows, 140, 0x5EED)
else:
    A = sk.SparseMatrix.convdiff3d_device(args.n, 100.0, 50.0, 25.0)
    S = sk.SketchOperator.subsampled_dct(A.rows, 240, 0x5EED)
b = sk.gaussian_vector(A.rows, 1)
j, br, rn = C.c_int64(), C.c_int(), C.c_double()
for rep in range(1):
    sk._check(sk._lib.sdr_krylov_run(ctx._h, A._h, S._h, b.ctypes.data_as(C.c_void_p), 2, 100, args.steps, 1e-14,
                                     None, None, None, None, C.byref(j), C.byref(br), C.byref(rn), None))
n = C.c_int64()
buf = np.zeros(8 * 1024, dtype=np.uint64)
sk._check(sk._lib.sdr_debug_trace(ctx._h, buf.ctypes.data_as(C.c_void_p), buf.size, C.byref(n)))
tr = buf[: n.value].reshape(-1, 16).astype(np.int64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
rel = (tr - t0) / 1e3  # us
rel[tr == 0] = np.nan
names = ["start", "prologue", "main", "combine", "pdl_wait"]
print(f"CTAs {len(tr)}; times in us from the first CTA start")
for k, nm in enumerate(names):
    col = rel[:, k]
    col = col[~np.isnan(col)]
    col = col[col >= 0]
    if len(col):
        print(f"  {nm:9s} n={len(col):4d} min {col.min():8.2f} median {np.median(col):8.2f} max {col.max():8.2f}")
d = rel[:, 2] - rel[:, 1]
print(f"  main-loop duration per CTA: min {np.nanmin(d):.2f} median {np.nanmedian(d):.2f} max {np.nanmax(d):.2f}")
