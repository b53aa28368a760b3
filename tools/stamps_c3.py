"""Device-clock timeline (SDR_TRACE=2 launch stamps, no host events in the
stream) of two systems of the C3 sequence: per-kernel durations, gaps, GPU
idle. Usage: SDR_TRACE=2 python tools/stamps_c3.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

assert os.environ.get("SDR_TRACE") == "2"
n = 1024
N = n * n
ctx = sk.default_context()
b0 = sk.gaussian_vector(N, 0x3000)
probs = []
for i in range(2):
    rel = 1e-3 * (2.0 * sk.uniform_stream(0x3100 + i, N) - 1.0)
    off, col, val = sk.gen_convdiff2d(n, 100.0 + 2 * i, 100.0 - 2 * i, 0.01 * i, rel)
    probs.append(sk.ProblemInstance(sk.SparseMatrix(N, N, off, col, val, ctx=ctx),
                                    b0 + 0.05 * sk.gaussian_vector(N, 0x3000 + i) if i else b0.copy()))
cfg = sk.SolverConfig(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact")
S = sk.SketchOperator.subsampled_dct(N, 140, cfg.sketch_seed, ctx=ctx)
sk.solve_sequence(probs, cfg, sketch=S)
path = "gpurun_out/stamps_c3.csv"
os.makedirs("gpurun_out", exist_ok=True)
sk._check(sk._lib.sdr_debug_stamps(ctx._h, path.encode()))
import time  # noqa: E402
t0 = time.perf_counter()
out = sk.solve_sequence(probs, cfg, sketch=S)
ctx.synchronize()
wall = time.perf_counter() - t0
sk._check(sk._lib.sdr_debug_stamps(ctx._h, path.encode()))
rows = [ln.strip().split(",") for ln in open(path).read().splitlines()[1:]]
rows = sorted(((nm, int(a), int(e)) for nm, a, e in rows if int(e) > 0), key=lambda x: x[1])
span = (rows[-1][2] - rows[0][1]) / 1e6
its = sum(r.iterations for r in out.reports)
print(f"{its} steps, wall {wall * 1e3:.1f} ms ({its / wall:.0f} steps/s), stamped span {span:.1f} ms")
dur = {}
for nm, a, e in rows:
    dur.setdefault(nm, []).append((e - a) / 1e3)
for nm, v in dur.items():
    print(f"  {nm:14s} n={len(v):5d} median {np.median(v):7.2f} us total {sum(v) / 1e3:7.2f} ms")
busy = sum(sum(v) for v in dur.values()) / 1e3
print(f"  stamped kernels busy {busy:.1f} ms of the {span:.1f} ms span")
gaps = [(a1 - e0) / 1e3 for (_, _, e0), (_, a1, _) in zip(rows, rows[1:])]
g = np.array(gaps)
print(f"  gaps: median {np.median(g):.2f} us, total {g[g > 0].sum() / 1e3:.2f} ms, >100us: {(g > 100).sum()} "
      f"({g[g > 100].sum() / 1e3:.2f} ms)")
