"""Device-clock stamps (SDR_TRACE=2, no host events in the stream) of one C2
solve: step-kernel durations and every gap > 50 us between stamped launches
(restarts). Usage: SDR_TRACE=2 python tools/stamps_c2.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

assert os.environ.get("SDR_TRACE") == "2"
ctx = sk.default_context()
A = sk.SparseMatrix.convdiff3d_device(128, 100.0, 50.0, 25.0)
import torch  # noqa: E402
b = torch.from_numpy(sk.gaussian_vector(A.rows, 1)).cuda()
cfg = sk.SolverConfig(m=100, k=20, t=2, s=240, tol=1e-8)
S = sk.SketchOperator.subsampled_dct(A.rows, 240, cfg.sketch_seed)
for _ in range(2):
    sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S)
path = "gpurun_out/stamps_c2.csv"
os.makedirs("gpurun_out", exist_ok=True)
sk._check(sk._lib.sdr_debug_stamps(ctx._h, path.encode()))
r = sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S)
ctx.synchronize()
sk._check(sk._lib.sdr_debug_stamps(ctx._h, path.encode()))
rows = [ln.strip().split(",") for ln in open(path).read().splitlines()[1:]]
rows = sorted(((nm, int(a), int(e)) for nm, a, e in rows if int(e) > 0), key=lambda x: x[1])
t0 = rows[0][1]
print(f"{r.report.iterations} it, report {r.report.seconds * 1e3:.2f} ms, stamped span {(rows[-1][2] - t0) / 1e6:.2f} ms")
for i in range(1, len(rows)):
    g = (rows[i][1] - rows[i - 1][2]) / 1e3
    if g > 50:
        print(f"  gap {g:8.1f} us at {(rows[i][1] - t0) / 1e3:9.1f} us: {rows[i - 1][0]} -> {rows[i][0]}")
dur = {}
for nm, a, e in rows:
    dur.setdefault(nm, []).append((e - a) / 1e3)
for nm, v in dur.items():
    print(f"  {nm:14s} n={len(v):5d} median {np.median(v):7.2f} us total {sum(v) / 1e3:7.2f} ms")
