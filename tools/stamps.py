"""Device-clock timeline of the step kernels (SDR_TRACE=2): durations of K1 /
K2 from first-CTA start to last-CTA end and the gaps between them, without
host events in the stream. Usage: SDR_TRACE=2 python tools/stamps.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

assert os.environ.get("SDR_TRACE") == "2"
ctx = sk.default_context()
A = sk.SparseMatrix.convdiff3d_device(128, 100.0, 50.0, 25.0)
b = sk.gaussian_vector(A.rows, 1)
cfg = sk.SolverConfig(m=100, k=20, t=2, s=240, tol=1e-8)
S = sk.SketchOperator.subsampled_dct(A.rows, 240, cfg.sketch_seed)
path = "gpurun_out/stamps.csv"
os.makedirs("gpurun_out", exist_ok=True)
for _ in range(2):
    sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S)
sk._check(sk._lib.sdr_debug_stamps(ctx._h, path.encode()))  # discard warm-up stamps
r = sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S)
sk._check(sk._lib.sdr_debug_stamps(ctx._h, path.encode()))
rows = [ln.strip().split(",") for ln in open(path).read().splitlines()[1:]]
rows = [(n, int(a), int(e)) for n, a, e in rows if int(e) > 0]
rows.sort(key=lambda x: x[1])
t0 = rows[0][1]
print(f"solve {r.report.iterations} it, {r.report.seconds*1e3:.2f} ms; stamped launches {len(rows)}, "
      f"span {(rows[-1][2]-t0)/1e6:.2f} ms")
dur = {}
for n, a, e in rows:
    dur.setdefault(n, []).append((e - a) / 1e3)
for n, v in dur.items():
    print(f"  {n:14s} n={len(v):4d} median {np.median(v):7.2f} us  mean {np.mean(v):7.2f}")
gaps = {}
for (n0, a0, e0), (n1, a1, e1) in zip(rows, rows[1:]):
    gaps.setdefault(f"{n0}->{n1}", []).append((a1 - e0) / 1e3)
for k, v in gaps.items():
    v = np.array(v)
    print(f"  gap {k:30s} n={len(v):4d} median {np.median(v):8.2f} us  p90 {np.percentile(v, 90):8.2f}")
st = np.array([a for n, a, e in rows if n == "spmv_arnoldi"])
d = np.diff(st) / 1e3
print(f"  step period (K1 start to next K1 start): median {np.median(d):.2f} us  (n={len(d)}, cycle restarts excluded: "
      f"{np.median(d[d < 200]):.2f})")
# GPU idle between consecutive stamped launches (K1/K2/sketch only; boundaries also run unstamped kernels)
idle = sum(max(0, a1 - e0) for (n0, a0, e0), (n1, a1, e1) in zip(rows, rows[1:])) / 1e6
print(f"  idle between stamped launches: {idle:.2f} ms of a {(rows[-1][2]-rows[0][1])/1e6:.2f} ms span")
big = sorted(((a1 - e0) / 1e3, n0, n1, (a1 - t0) / 1e3) for (n0, a0, e0), (n1, a1, e1) in zip(rows, rows[1:]))[-8:]
print("  largest gaps (us, after, before, at us):", [(round(g), x, y, round(t)) for g, x, y, t in big])
