"""Host LAPACK probe on the GPU box: 120 x 120 SVD / Schur / Hessenberg times at
1..8 OpenBLAS threads (the restart pencil's host cost). Usage: python tools/lapack_probe.py"""
import sys, os; sys.path.insert(0, os.getcwd())
import time, numpy as np, scipy.linalg as sl
print('cpus', os.cpu_count(), open('/proc/cpuinfo').read().split('model name')[1].split('\n')[0])
rng=np.random.default_rng(0)
R=np.triu(rng.standard_normal((120,120))); C=rng.standard_normal((120,120))
def t(f, n=20):
    f(); t0=time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter()-t0)/n*1e3
from threadpoolctl import threadpool_limits
for th in (1, 2, 4, 8):
    with threadpool_limits(th):
        print(th, 'gesdd R', round(t(lambda: sl.svd(R, full_matrices=False, lapack_driver='gesdd')),3),
              'gesvd R', round(t(lambda: sl.svd(R, full_matrices=False, lapack_driver='gesvd')),3),
              'schur', round(t(lambda: sl.schur(C, output='real')),3),
              'eigvals', round(t(lambda: sl.eigvals(C)),3),
              'hess', round(t(lambda: sl.hessenberg(C, calc_q=True)),3))
