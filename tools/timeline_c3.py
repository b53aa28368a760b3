"""Device timeline (timed launches) of the first two systems of the C3
sequence: per-kernel totals and the largest gaps. Usage: python tools/timeline_c3.py"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402

n = 1024
N = n * n
ctx = sk.default_context()
b0 = sk.gaussian_vector(N, 0x3000)
probs = []
for i in range(2):
    rel = 1e-3 * (2.0 * sk.uniform_stream(0x3100 + i, N) - 1.0)
    off, col, val = sk.gen_convdiff2d(n, 100.0 + 2 * i, 100.0 - 2 * i, 0.01 * i, rel)
    A = sk.SparseMatrix(N, N, off, col, val, ctx=ctx)
    b = b0 + 0.05 * sk.gaussian_vector(N, 0x3000 + i) if i else b0.copy()
    probs.append(sk.ProblemInstance(A, b))
cfg = sk.SolverConfig(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact")
S = sk.SketchOperator.subsampled_dct(N, 140, cfg.sketch_seed, ctx=ctx)
sk.solve_sequence(probs, cfg, sketch=S)
ctx.set_timing(True)
ctx.timing_reset()
out = sk.solve_sequence(probs, cfg, sketch=S)
path = "gpurun_out/timeline_c3.csv"
os.makedirs("gpurun_out", exist_ok=True)
sk._check(sk._lib.sdr_debug_timeline(ctx._h, path.encode()))
ctx.set_timing(False)
rows = []
with open(path) as fh:
    next(fh)
    for ln in fh:
        name, a, e = ln.strip().split(",")
        rows.append((name, float(a), float(e)))
rows.sort(key=lambda r: r[1])
span = rows[-1][2] - rows[0][1]
busy = collections.defaultdict(lambda: [0, 0.0])
for nme, a, e in rows:
    busy[nme][0] += 1
    busy[nme][1] += e - a
print(f"iterations {[r.iterations for r in out.reports]}, span {span/1e3:.2f} ms, "
      f"kernel time {sum(v[1] for v in busy.values())/1e3:.2f} ms")
print({k: (v[0], round(v[1] / 1e3, 3)) for k, v in sorted(busy.items(), key=lambda kv: -kv[1][1])})
gaps = collections.defaultdict(lambda: [0, 0.0])
for (n0, a0, e0), (n1, a1, e1) in zip(rows, rows[1:]):
    g = a1 - e0
    if g > 0:
        gaps[f"{n0} -> {n1}"][0] += 1
        gaps[f"{n0} -> {n1}"][1] += g
print("gaps (count, ms):", {k: (v[0], round(v[1] / 1e3, 3)) for k, v in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:12]})
