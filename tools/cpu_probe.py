"""Host CPU probe: single-thread dgemm rate and small LAPACK kernels (for the
host-side harmonic/QR cost model)."""
import os
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import time
import numpy as np
import scipy.linalg as sl

rng = np.random.default_rng(0)


def t(f, n=5):
    f()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e3


A = rng.standard_normal((512, 512))
ms = t(lambda: A @ A)
print(f"dgemm 512: {ms:.2f} ms = {2*512**3/ms/1e6:.1f} GFLOP/s")
B = rng.standard_normal((240, 120))
print(f"gesdd 240x120: {t(lambda: sl.svd(B, full_matrices=False, lapack_driver='gesdd')):.2f} ms")
print(f"qr 240x120: {t(lambda: sl.qr(B, mode='economic')):.2f} ms")
C = rng.standard_normal((120, 120))
print(f"svd 120x120: {t(lambda: sl.svd(C)):.2f} ms")
S = C @ C.T
print(f"schur sym-ish 120: {t(lambda: sl.schur(S + 0.1 * C, output='real')):.2f} ms")
print(f"hessenberg 120: {t(lambda: sl.hessenberg(C)):.2f} ms")
