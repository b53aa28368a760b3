"""Device timeline of one C2 solve (timed launches): per-kernel totals, gaps
between consecutive launches, and the GPU-idle share.
Usage: python tools/timeline.py [--n 128] [--csv gpurun_out/timeline.csv]"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--csv", default="gpurun_out/timeline.csv")
args = ap.parse_args()
ctx = sk.default_context()
A = sk.SparseMatrix.convdiff3d_device(args.n, 100.0, 50.0, 25.0)
b = sk.gaussian_vector(A.rows, 1)
cfg = sk.SolverConfig(m=100, k=20, t=2, s=240, tol=1e-8)
S = sk.SketchOperator.subsampled_dct(A.rows, 240, cfg.sketch_seed)
for _ in range(2):
    sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S)
ctx.set_timing(True)
ctx.timing_reset()
r = sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S)
os.makedirs(os.path.dirname(args.csv) or ".", exist_ok=True)
sk._check(sk._lib.sdr_debug_timeline(ctx._h, args.csv.encode()))
ctx.set_timing(False)
rows = []
with open(args.csv) as fh:
    next(fh)
    for line in fh:
        n, a, e = line.strip().split(",")
        rows.append((n, float(a), float(e)))
rows.sort(key=lambda x: x[1])
span = rows[-1][2] - rows[0][1]
busy = sum(e - a for _, a, e in rows)
print(f"solve {r.report.iterations} it, report {r.report.seconds*1e3:.2f} ms; timeline span {span/1e3:.2f} ms, "
      f"kernels {busy/1e3:.2f} ms ({100*busy/span:.1f}%)")
tot = collections.defaultdict(lambda: [0, 0.0])
gaps = collections.defaultdict(lambda: [0, 0.0])
for i, (n, a, e) in enumerate(rows):
    tot[n][0] += 1
    tot[n][1] += e - a
    if i:
        g = a - rows[i - 1][2]
        key = f"{rows[i-1][0]} -> {n}"
        gaps[key][0] += 1
        gaps[key][1] += max(g, 0.0)
print("kernel totals (ms):", {k: (v[0], round(v[1] / 1e3, 3)) for k, v in sorted(tot.items(), key=lambda x: -x[1][1])})
print("largest gap classes (count, total ms, mean us):")
for k, v in sorted(gaps.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {k:40s} {v[0]:5d} {v[1]/1e3:8.3f} {v[1]/max(v[0],1):8.2f}")
big = sorted(((a - rows[i - 1][2], rows[i - 1][0], n, a) for i, (n, a, e) in enumerate(rows) if i), reverse=True)[:10]
print("top single gaps (us, after -> before, at us):", [(round(g, 1), x, y, round(t)) for g, x, y, t in big])
