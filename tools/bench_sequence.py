"""C3 (BASELINE): a 20-system recycling sequence on one GPU.
N = 1024^2 2-D convection-diffusion, system i: beta = (100+2i, 100-2i), shift
0.01*i, diagonal perturbation of relative size 1e-3 (uniform stream seed
0x3100+i), b_i = b_0 + 0.05 xi_i (gaussian seeds 0x3000 / 0x3000+i),
m=50 k=20 t=2 s=140 tol=1e-8, variant exact (refresh on every matrix change).
Same seeds and construction as tests/golden/make_golden.py c3_small.
Prints one JSON line: total Arnoldi steps / sequence wall time, with b and
x in HBM (`value`) and through host numpy arrays (`e2e`; --host: only that).
Usage: python tools/bench_sequence.py [--n 1024] [--count 20] [--steps 2] [--host]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--count", type=int, default=20)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--host", action="store_true", help="right-hand sides and solutions in host memory (e2e only)")
args = ap.parse_args()
n, count = args.n, args.count
N = n * n
ctx = sk.default_context()


def uniform_stream(seed, length):
    """Rng::uniform stream (rng.hpp:32) through the library's generator."""
    return sk.uniform_stream(seed, length)


t0 = time.time()
b0 = sk.gaussian_vector(N, 0x3000)
probs = []
for i in range(count):
    rel = 1e-3 * (2.0 * uniform_stream(0x3100 + i, N) - 1.0)
    off, col, val = sk.gen_convdiff2d(n, 100.0 + 2 * i, 100.0 - 2 * i, 0.01 * i, rel)
    A = sk.SparseMatrix(N, N, off, col, val, ctx=ctx)
    b = b0 + 0.05 * sk.gaussian_vector(N, 0x3000 + i) if i else b0.copy()
    probs.append(sk.ProblemInstance(A, b))
setup_s = time.time() - t0
cfg = sk.SolverConfig(m=50, k=20, t=2, s=140, tol=1e-8, variant="exact")
S = sk.SketchOperator.subsampled_dct(N, 140, cfg.sketch_seed, ctx=ctx)
probs_host = probs
outs = None
if not args.host:
    # value: b and x resident in HBM (as bench.py's `value`); e2e below with host arrays
    import torch
    probs = [sk.ProblemInstance(p.matrix, torch.from_numpy(p.rhs).cuda()) for p in probs_host]
    outs = [torch.zeros(N, dtype=torch.float64, device="cuda") for _ in probs]


def run(ps, o):
    walls, iters, out = [], 0, None
    for _ in range(args.warmup):
        sk.solve_sequence(ps, cfg, sketch=S, outs=o)
    ctx.synchronize()
    for _ in range(args.steps):
        t1 = time.perf_counter()
        out = sk.solve_sequence(ps, cfg, sketch=S, outs=o)
        ctx.synchronize()
        walls.append(time.perf_counter() - t1)
        iters += sum(r.iterations for r in out.reports)
    return walls, iters, out


walls, iters, out = run(probs, outs)
total = sum(walls)
e2e = None
if not args.host:
    w2, i2, _ = run(probs_host, None)
    e2e = {"value": i2 / sum(w2), "unit": "steps/s", "h2d_bytes_per_step": 8 * N * count,
           "d2h_bytes_per_step": 8 * N * count, "path": "solve_sequence with host (pageable numpy) b and x"}
phases = {}
for r in out.reports:
    for k, v in r.phases.items():
        phases[k] = phases.get(k, 0.0) + v
line = {
    "metric": "gmres_sdr_arnoldi_steps_per_s", "value": iters / total, "unit": "steps/s", "n_gpus": 1,
    "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
    "dtype": "f64", "data": "synthetic (BASELINE C3 construction, seeded)",
    "config": {"workload": "c3", "N": N, "systems": count, "m": 50, "k": 20, "t": 2, "s": 140, "tol": 1e-8,
               "variant": "exact", "storage": probs[0].matrix.storage},
    "residency": "host b / x" if args.host else "b / x in HBM",
    "e2e": e2e,
    "sequence": {"iterations": [r.iterations for r in out.reports], "status": [r.status for r in out.reports],
                 "cycles": [r.cycles for r in out.reports],
                 "final_relative_residual": [r.final_relative_residual for r in out.reports],
                 "wall_s": [round(w, 4) for w in walls], "setup_s": round(setup_s, 2),
                 "phases_ms": {k: round(v, 2) for k, v in sorted(phases.items(), key=lambda kv: -kv[1])}},
}
print(json.dumps(line), flush=True)
