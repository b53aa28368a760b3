"""Sparse-sign sketch apply timing (CUDA events) and an ncu target.
Usage: python tools/sparse_sign_probe.py [--n 33554432] [--s 120] [--reps 20]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 25)
ap.add_argument("--s", type=int, default=120)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
ctx = sk.default_context()
S = sk.SketchOperator.sparse_sign(args.n, args.s, 0x5EED, 8, ctx=ctx)
x = torch.randn(args.n, dtype=torch.float64, device="cuda")
S.apply(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    S.apply(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.reps
print(f"sparse sign n={args.n} s={args.s}: {ms * 1e3:.1f} us per apply (incl. host round trip), "
      f"{8 * args.n / (ms * 1e-3) / 1e9:.0f} GB/s of x")
