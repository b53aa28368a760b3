"""GMRES-SDR vs the device classical restarted GMRES on the
same B200: C2 (128^3 convection-diffusion, m=100, tol 1e-8) and the grid
family of acceptance criteria 6/8 (50 rhs, 103^2 Neumann grid, m=100,
tol 1e-6). Reports steps/s, time to solution and inner products of both.
Usage: python tools/bench_baseline.py [--n 128] [--family]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_14206_b200 as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--restarts", type=int, default=10)
ap.add_argument("--family", action="store_true")
args = ap.parse_args()
ctx = sk.default_context()
out = {}


def timed(fn, reps=2):
    fn()
    ctx.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        r = fn()
    ctx.synchronize()
    return r, (time.perf_counter() - t) / reps


n = args.n
A = sk.SparseMatrix.convdiff3d_device(n, 100.0, 50.0, 25.0)
b = sk.gaussian_vector(n ** 3, 1)
sdr, t_sdr = timed(lambda: sk.solve(A, b, sk.SolverConfig(m=100, k=20, t=2, s=240, tol=1e-8)))
bl, t_bl = timed(lambda: sk.baseline_gmres(A, b, sk.BaselineConfig(m=100, tol=1e-8, max_restarts=args.restarts)), 1)
out["c2"] = {
    "gmres_sdr": {"status": sdr.report.status, "steps": sdr.report.iterations, "seconds": t_sdr,
                  "steps_per_s": sdr.report.iterations / t_sdr,
                  "inner_products": sdr.report.counters["inner_products"],
                  "final_relative_residual": sdr.report.final_relative_residual},
    "baseline": {"status": bl.report.status, "steps": bl.report.iterations, "seconds": t_bl,
                 "steps_per_s": bl.report.iterations / t_bl, "inner_products": bl.report.counters["inner_products"],
                 "final_relative_residual": bl.report.final_relative_residual,
                 "true_residuals": bl.report.true_residuals[:12]},
}
if args.family:
    from oracle import pyoracle as O  # test-side generator of the acceptance operator only
    M = O.gen_neumann(103, 1e-4)
    off, col, val = M.csr()
    G = sk.SparseMatrix(M.rows, M.cols, off, col, val)
    rhs = [sk.gaussian_vector(M.rows, 2026 + i) for i in range(50)]
    cfg = sk.SolverConfig(m=100, t=2, k=20, s=1200, tol=1e-6, max_restarts=10)
    seq, t_seq = timed(lambda: sk.solve_sequence([sk.ProblemInstance(G, x, target_tol=1e-6) for x in rhs], cfg,
                                                 shared_matrix=True), 1)
    bcfg = sk.BaselineConfig(m=100, tol=1e-6, max_restarts=10)
    bls, t_bls = timed(lambda: [sk.baseline_gmres(G, x, bcfg) for x in rhs], 1)
    out["grid_family"] = {
        "gmres_sdr": {"converged": sum(r.status == "converged" for r in seq.reports), "seconds": t_seq,
                      "steps": sum(r.iterations for r in seq.reports),
                      "inner_products": sum(r.counters["inner_products"] for r in seq.reports)},
        "baseline": {"converged": sum(r.report.status == "converged" for r in bls), "seconds": t_bls,
                     "steps": sum(r.report.iterations for r in bls),
                     "inner_products": sum(r.report.counters["inner_products"] for r in bls)},
    }
print(json.dumps(out))
