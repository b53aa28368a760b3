import ctypes as C, sys, numpy as np
sys.path.insert(0, '.')
import paper_2311_14206_b200 as sk
L = sk._lib
L.sdr_debug_norm2.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_double)]
ctx = sk.default_context()
for n in (60, 1000, 100000, 3000000):
    x = np.ones(n)
    o = C.c_double()
    sk._check(L.sdr_debug_norm2(ctx._h, x.ctypes.data_as(C.c_void_p), n, C.byref(o)))
    print(n, o.value)
