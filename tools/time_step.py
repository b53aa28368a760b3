"""Isolated CUDA-event timing of the C2 step kernels (sdr_debug_time_step):
K1 (SpMV + window dots) and K2 (fused update + SRDCT), back-to-back relaunches.
Usage: [SDR_K2_VARIANT=v] python tools/time_step.py [--n 128] [--reps 50]"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--repeat", type=int, default=3)
args = ap.parse_args()
A = sk.SparseMatrix.convdiff3d_device(args.n, 100.0, 50.0, 25.0)
b = sk.gaussian_vector(A.rows, 1)
S = sk.SketchOperator.subsampled_dct(A.rows, 240, 0x5EED)
for _ in range(args.repeat):
    k1, k2 = C.c_double(), C.c_double()
    sk._check(sk._lib.sdr_debug_time_step(A.ctx._h, A._h, S._h, b.ctypes.data_as(C.c_void_p), 2, 100, 20, args.reps,
                                          C.byref(k1), C.byref(k2)))
    print(f"variant {os.environ.get('SDR_K2_VARIANT', '0')}: K1 {k1.value:.2f} us  K2 {k2.value:.2f} us")
