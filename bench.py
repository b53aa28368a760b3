"""GMRES-SDR benchmark (BASELINE.json metric: Arnoldi steps/s & time-to-solution,
achieved HBM GB/s vs peak).

One bench "step" = one complete GMRES-SDR solve of the workload (fresh recycle
space each time) — every Arnoldi step, host least-squares, verification and
harmonic recycle update inside the timed region. value = total Arnoldi steps
of all ranks / max-over-ranks device time.

Workloads (BASELINE.json configs, synthetic data per their generators):
  c2 (default, N=1): 3D 7-point −Δu+β·∇u on 128³, β=(100,50,25), b=gaussian_vector(N,1),
                     m=100 k=20 t=2 s=240 tol=1e-8, SRDCT seed 0x5eed.
  With --gpus N>1 each rank owns a 128³ z-slab of a 128×128×(128·N) grid (weak scaling).
  c5:               512³, β=(200,100,50), b seed 3, m=50 k=10 t=2 s=120 tol=1e-7, sparse sign ζ=8.

--impl reference times the CPU oracle (the reference cannot be compiled here:
Eigen/FFTW/LAPACKE absent — DESIGN.md §oracle) on the same workload: a bounded
sample of init_krylov + Arnoldi steps per bench step, single-threaded like the reference.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    "c2": dict(n=128, beta=(100.0, 50.0, 25.0), seed=1, m=100, k=20, t=2, s=240, tol=1e-8, sketch="srdct"),
    "c5": dict(n=512, beta=(200.0, 100.0, 50.0), seed=3, m=50, k=10, t=2, s=120, tol=1e-7, sketch="sparse_sign"),
}
METRIC = "gmres_sdr_arnoldi_steps_per_s"


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed
    region through NVML (the library nvidia-smi queries; polling in-process
    avoids a competing nvidia-smi client contending for the driver)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, device, period=0.1):
        self.device = device
        self.period = period
        self.samples = []
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _sample(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append((sm, rs))

    def _run(self):
        while not self._stop.wait(self.period):
            try:
                self._sample()
            except Exception:
                break

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for _, rs in self.samples for name, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def bytes_per_step(N, a_bytes, t):
    """B_step = bytes(A) + 8 N (4 + 2t), with bytes(A) the
    operator storage one SpMV streams (CSR in the reference: 12 nnz + 4 (N+1);
    here SELL-DIA 8 B per stored entry, or SELL-32 12 B; A.storage["bytes"])."""
    return a_bytes + 8 * N * (4 + 2 * t)


def kernel_bytes(N, a_bytes, t, sketch):
    """Algorithmic bytes per launch of each hot kernel."""
    return {
        "spmv_arnoldi": a_bytes + 8 * N * (2 + (t - 1)),          # A, x, y write, t-1 window reads
        "update": 8 * N * (1 + t) + 8 * N,                        # y + t window reads, w write
        "update_sketch": 8 * N * (1 + t) + 8 * N + N // 8,        # fused update + SRDCT: the update's bytes (+ sign bits)
        "sketch": 8 * N + (N // 8 if sketch == "srdct" else 0),  # one read of w (+ sign bits)
    }


def run_reference(args, wl, rank, world):
    """CPU oracle on a bounded sample of the same workload (rank 0 only)."""
    if rank != 0:
        return None
    from oracle import pyoracle as O
    n = wl["n"]
    N = n ** 3
    t0 = time.time()
    A = O.gen_convdiff3d(n, *wl["beta"])
    b = O.gaussian_vector(N, wl["seed"])
    S = (O.SketchOperator.subsampled_dct(N, wl["s"], 0x5EED) if wl["sketch"] == "srdct"
         else O.SketchOperator.sparse_sign(N, wl["s"], 0x5EED, 8))
    setup = time.time() - t0
    steps_per_sample = int(os.environ.get("SDR_REF_STEPS", "8"))
    for _ in range(args.warmup and 1):
        O.run_arnoldi(A, b, S, wl["t"], 1, steps=1)
    times = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        st = O.run_arnoldi(A, b, S, wl["t"], steps_per_sample, steps=steps_per_sample)
        times.append(time.perf_counter() - t1)
        assert st.j == steps_per_sample
    total = sum(times)
    value = steps_per_sample * args.steps / total
    sample = (f"init_krylov + {steps_per_sample} arnoldi_step of workload {args.config} (N={N}) per bench step "
              f"(oracle C++ restatement, 1 thread; reference unbuildable here)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "N": N, "nnz": A.nnz, "m": wl["m"], "k": wl["k"], "t": wl["t"],
                   "s": wl["s"], "sketch": wl["sketch"]},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": setup,
    }
    return line


_JSON_OUT = None


def emit(line):
    """The one JSON line on the real stdout (library / NCCL banners that write to
    fd 1 during the run are sent to stderr, see __main__)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    wl = WORKLOADS[args.config]
    rank, world, local = dist_env()

    if args.impl == "reference":
        line = run_reference(args, wl, rank, world)
        if line is not None:
            emit(line)
        return

    import torch
    torch.cuda.set_device(local)
    import paper_2311_14206_b200 as sk

    # SDR_BENCH_DIST=1 takes the multi-GPU code path even on one rank (one-rank
    # NCCL communicator): a check of the torchrun / NCCL plumbing on one GPU
    if world > 1 or os.environ.get("SDR_BENCH_DIST") == "1":
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        idbuf = [sk.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(idbuf, src=0)
        ctx = sk.Context(local, rank, world, idbuf[0])
    else:
        dist = None
        ctx = sk.Context(local)

    n = wl["n"]
    nz = n * world if args.config == "c2" else n
    z0, z1 = (rank * n, (rank + 1) * n) if args.config == "c2" else (nz * rank // world, nz * (rank + 1) // world)
    A = sk.SparseMatrix.convdiff3d_device(n, *wl["beta"], z_begin=z0, z_end=z1, ctx=ctx, ny=n, nz=nz)
    N = A.rows
    nloc = A.local_rows
    # b = gaussian_vector(N, seed): every rank draws the same stream and keeps its block
    b_full = sk.gaussian_vector(N, wl["seed"]) if world == 1 else sk.gaussian_vector(N, wl["seed"])[A.row_begin:A.row_begin + nloc]
    b_host = torch.from_numpy(np.ascontiguousarray(b_full)).pin_memory()
    b_dev = b_host.to(f"cuda:{local}")
    S = (sk.SketchOperator.subsampled_dct(N, wl["s"], 0x5EED, ctx=ctx) if wl["sketch"] == "srdct"
         else sk.SketchOperator.sparse_sign(N, wl["s"], 0x5EED, 8, ctx=ctx))
    cfg = sk.SolverConfig(m=wl["m"], k=wl["k"], t=wl["t"], s=wl["s"], tol=wl["tol"])
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")

    def barrier():
        if dist is not None:
            dist.barrier()

    def one(b, host=False):
        space = sk.RecycleSpace(ctx)
        r = sk.solve(A, b, cfg, space=space, sketch=S)
        return r

    for _ in range(args.warmup):
        r = one(b_dev)
    # ---- timed region: device-resident input (value)
    barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    reports = []
    walls = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            tw = time.perf_counter()
            r = one(b_dev)
            walls.append(1e3 * (time.perf_counter() - tw))
            iters += r.report.iterations
            reports.append(r.report)
        ev1.record(stream)
        ev1.synchronize()
    ctx.synchronize()
    torch.cuda.synchronize()
    barrier()
    launches = ctx.launches - launches0
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms, float(iters)], dtype=torch.float64)
        gathered = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, t)
        ms = max(float(g[0]) for g in gathered)
    # Every rank takes the same (global) Arnoldi steps, each over its own 128³
    # slab: whole-job throughput counts slab-steps, iterations x world / time.
    value = (iters * world) / (ms / 1e3)

    # ---- e2e through the public API with host buffers (H2D of b, D2H of x inside)
    e2e_iters = 0
    e2e_walls = []
    x_host = torch.empty(nloc, dtype=torch.float64).pin_memory()  # the user's pinned result buffer
    for _ in range(max(1, args.warmup // 2)):  # warm the host-buffer path (first-touch staging)
        sk.solve(A, b_host.numpy(), cfg, space=sk.RecycleSpace(ctx), sketch=S, out=x_host.numpy())
    ctx.synchronize()
    barrier()
    t_e2e0 = time.perf_counter()
    for _ in range(args.steps):
        tw = time.perf_counter()
        space = sk.RecycleSpace(ctx)
        r = sk.solve(A, b_host.numpy(), cfg, space=space, sketch=S, out=x_host.numpy())
        e2e_iters += r.report.iterations
        e2e_walls.append(1e3 * (time.perf_counter() - tw))
    ctx.synchronize()
    e2e_s = time.perf_counter() - t_e2e0
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, t)
        e2e_s = max(float(g[0]) for g in gathered)
    e2e_value = e2e_iters * world / e2e_s

    # ---- per-kernel roofline from CUDA events on the library stream (one instrumented solve)
    ctx.set_timing(True)
    ctx.timing_reset()
    rt = one(b_dev)
    ctx.synchronize()
    ktimes = {k: ctx.timing(k) for k in ("spmv_arnoldi", "update", "sketch", "update_sketch", "sketch_fold", "sketch_side",
                                         "tallskinny", "recycle_gemm", "col_norms", "correction", "residual",
                                         "copy_norm", "allreduce", "halo", "axpy")}
    ctx.set_timing(False)
    kb = kernel_bytes(nloc, A.storage["bytes"], wl["t"], wl["sketch"])
    peak, peak_kind = measured_peak()
    kern = {}
    for name, (cnt, tot) in ktimes.items():
        if cnt:
            d = {"launches": cnt, "avg_us": 1e3 * tot / cnt, "share": 0.0}
            if name in kb:
                d["GBps"] = kb[name] / (tot / cnt * 1e-3) / 1e9
                d["frac"] = d["GBps"] / peak
            kern[name] = d
    tot_all = sum(v["avg_us"] * v["launches"] for v in kern.values())
    for v in kern.values():
        v["share"] = v["avg_us"] * v["launches"] / tot_all if tot_all else 0.0
    dom = max((k for k in kern if k in kb), key=lambda k: kern[k]["avg_us"] * kern[k]["launches"])
    step_us = sum(kern[k]["avg_us"] for k in kb if k in kern)
    step_bytes = bytes_per_step(nloc, A.storage["bytes"], wl["t"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as fh:
            traffic = json.load(fh).get(dom)
    except Exception:
        pass
    # the dominant kernel's launch duration without the per-launch event
    # instrumentation of the solve above: CUDA events around back-to-back
    # relaunches of a mid-cycle step's K1 / K2 on this workload (idempotent)
    iso = None
    if world == 1 and wl["sketch"] == "srdct" and dom in ("spmv_arnoldi", "update_sketch"):
        import ctypes as C
        k1, k2 = C.c_double(), C.c_double()
        b_np = np.ascontiguousarray(b_full)
        sk._check(sk._lib.sdr_debug_time_step(ctx._h, A._h, S._h, b_np.ctypes.data_as(C.c_void_p), wl["t"], wl["m"],
                                              20, 50, C.byref(k1), C.byref(k2)))
        iso = {"spmv_arnoldi": k1.value, "update_sketch": k2.value}
    dom_us = iso[dom] if iso else kern[dom]["avg_us"]
    dom_gbps = kb[dom] / (dom_us * 1e-6) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": dom_gbps, "peak": peak, "unit": "GB/s",
                "frac": dom_gbps / peak, "traffic": traffic, "peak_source": peak_kind,
                "bytes_per_launch": kb[dom], "launch_us": dom_us,
                "method": ("CUDA events around 50 back-to-back launches of the step kernel (C2 operator, mid-cycle "
                           "step j = 20)" if iso else "CUDA events around each launch of one instrumented solve"),
                "in_solve_event_us": kern[dom]["avg_us"],
                "isolated_us": iso,
                "isolated_frac": ({k: kb[k] / (v * 1e-6) / 1e9 / peak for k, v in iso.items()} if iso else None),
                "arnoldi_step": {"bytes": step_bytes, "us": step_us, "GBps": step_bytes / (step_us * 1e-6) / 1e9,
                                 "frac": step_bytes / (step_us * 1e-6) / 1e9 / peak,
                                 "timer": "sum of per-launch CUDA events in one instrumented solve"}}
    # the step as it runs inside a solve: device-clock stamps (no host events
    # in the stream), median interval between consecutive K1 starts
    try:
        import tempfile
        sk._check(sk._lib.sdr_ctx_set_stamps(ctx._h, 1))
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "stamps.csv").encode()
            sk._check(sk._lib.sdr_debug_stamps(ctx._h, path))  # reset
            one(b_dev)
            ctx.synchronize()
            sk._check(sk._lib.sdr_debug_stamps(ctx._h, path))
            starts = sorted(int(ln.split(",")[1]) for ln in open(path.decode()).read().splitlines()[1:]
                            if ln.startswith("spmv_arnoldi,") and int(ln.split(",")[2]) > 0)
        sk._check(sk._lib.sdr_ctx_set_stamps(ctx._h, 0))
        d = np.diff(np.array(starts, dtype=np.float64)) / 1e3
        med = float(np.median(d))
        per = float(np.median(d[d < 2.0 * med]))  # restart boundaries excluded
        roofline["arnoldi_step_pipelined"] = {"bytes": step_bytes, "period_us": per,
                                              "GBps": step_bytes / (per * 1e-6) / 1e9,
                                              "frac": step_bytes / (per * 1e-6) / 1e9 / peak,
                                              "timer": "device %globaltimer launch stamps in one solve: median "
                                                       "interval between consecutive K1 starts (restarts excluded)"}
    except Exception as e:  # measurement only
        print(f"step period measurement skipped: {e}", file=sys.stderr)
    if iso:
        iso_us = iso["spmv_arnoldi"] + iso["update_sketch"]
        roofline["arnoldi_step_isolated"] = {"bytes": step_bytes, "us": iso_us,
                                             "GBps": step_bytes / (iso_us * 1e-6) / 1e9,
                                             "frac": step_bytes / (iso_us * 1e-6) / 1e9 / peak}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        class A2:
            steps = 2
            warmup = 0
            config = args.config
        os.environ.setdefault("SDR_REF_STEPS", "8")
        ref = run_reference(A2, wl, 0, 1)
        cpu_baseline = dict(ref["cpu_baseline"])
        cpu_baseline["value"] = ref["value"]

    if rank == 0:
        rep = reports[-1]
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE generators, seeded)",
            "config": {"workload": args.config, "N": N, "N_per_gpu": nloc, "nnz": A.nnz, "storage": A.storage, "m": wl["m"], "k": wl["k"],
                       "t": wl["t"], "s": wl["s"], "tol": wl["tol"], "sketch": wl["sketch"],
                       "parallelism": f"zslab{world}", "l2": "inputs > L2 per solve (V basis 1.7 GB)"},
            "time_to_solution_ms": ms / args.steps,
            "solve": {"status": rep.status, "iterations": rep.iterations, "cycles": rep.cycles,
                      "final_relative_residual": rep.final_relative_residual,
                      "wall_ms": [round(v, 2) for v in walls], "e2e_wall_ms": [round(v, 2) for v in e2e_walls],
                      "internal_ms": [round(1e3 * rr.seconds, 2) for rr in reports],
                      "phases_ms": {k: round(v, 3) for k, v in rep.phases.items()}},
            "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": 8 * nloc, "d2h_bytes_per_step": 8 * nloc},
            "roofline": roofline,
            "kernels": kern,
            "cpu_baseline": cpu_baseline,
            "clocks": clk.summary(),
            "gpu_launches": launches,
        }
        emit(line)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    # keep stdout for the JSON line alone: fd 1 points at stderr while the
    # workload runs (NCCL prints its version banner to stdout on rank 0)
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    main()
