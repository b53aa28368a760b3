import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, os, numpy as np, scipy.linalg as sl
import paper_2311_14206_b200 as sk
print('cpus', os.cpu_count(), open('/proc/cpuinfo').read().split('model name')[1].split('\n')[0])
rng=np.random.default_rng(0)
A=rng.standard_normal((240,120)); C=rng.standard_normal((120,120))
def t(f, n=5):
    f(); t0=time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter()-t0)/n*1e3
print('gesdd', t(lambda: sl.svd(A, full_matrices=False, lapack_driver='gesdd')))
print('schur', t(lambda: sl.schur(C, output='real')))
SW=rng.standard_normal((240,120)); SAW=rng.standard_normal((240,120))
print('sdr_harmonic', t(lambda: sk.harmonic_pairs(SAW, SW, 20)))
