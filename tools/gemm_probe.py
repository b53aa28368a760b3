"""Recycle-product kernels (k_tsgemm vs k_rgemm) at n = 2^25, 60 inputs: ms and TB/s."""
import sys, ctypes as C; sys.path.insert(0, '.')
import torch, paper_2311_14206_b200 as sk
n, k1, k2 = 1 << 25, 50, 10
ctx = sk.default_context()
A1 = torch.randn(k1, n, dtype=torch.float64, device='cuda')
A2 = torch.randn(k2, n, dtype=torch.float64, device='cuda')
for nout in (10, 20):
    B = torch.randn(nout, k1 + k2, dtype=torch.float64, device='cuda')
    Cm = torch.empty(nout, n, dtype=torch.float64, device='cuda')
    nr = (C.c_double * nout)()
    for kern in (0, 1):
        def run():
            sk._check(sk._lib.sdr_debug_block_product(ctx._h, kern, n, C.c_void_p(A1.data_ptr()), n, k1, C.c_void_p(A2.data_ptr()), n, k2,
                                                      C.c_void_p(B.data_ptr()), nout, C.c_void_p(Cm.data_ptr()), n, nr))
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): run()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        gb = 8 * n * (k1 + k2 + nout) / 1e9
        print(f"nout {nout} kernel {'tsgemm' if kern == 0 else 'rgemm'}: {ms:.2f} ms, {gb / ms:.2f} TB/s")
