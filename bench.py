"""GMRES-SDR benchmark (BASELINE.json metric: Arnoldi steps/s & time-to-solution,
achieved HBM GB/s vs peak, 1/2/4/8 GPU).

One bench "step" = one complete GMRES-SDR solve of the workload to its
tolerance (fresh recycle space each time): every Arnoldi step, host least
squares, verification and harmonic recycle update inside the timed region.
value = Arnoldi steps of the (global) solve / max-over-ranks device time;
time_to_solution_ms = device time per solve.

Workloads (BASELINE.json configs, synthetic data from their generators):
  c5 (default): 3D 7-point -Δu+β·∇u on 512³ (N = 134,217,728), β=(200,100,50),
                b = gaussian_vector(N, 3), m=50 k=10 t=2 s=120 tol=1e-7, sparse
                sign ζ=8 (seed 0x5eed). max_restarts raised from the reference
                default 10 to 100 so the solve reaches 1e-7 (33 cycles).
  c2:           128³ (N = 2,097,152), β=(100,50,25), b seed 1, m=100 k=20 t=2 s=240
                tol=1e-8, SRDCT seed 0x5eed (reference default sketch).
--gpus N (N > 1): the same global problem, z-slab row partition over N ranks
(strong scaling); without torchrun's env, bench.py relaunches itself under
torch.distributed.run with N processes (NCCL_DEBUG=INFO).

--impl reference: the CPU oracle (the reference cannot be compiled here:
Eigen/FFTW/LAPACKE absent — DESIGN.md §6) on the same workload, rank 0 only:
init_krylov once, then one solve_cycle step (arnoldi_step + QR append + LS
solve, solver.hpp:165-179) per bench step, single-threaded like the reference.
"""
import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    "c5": dict(n=512, beta=(200.0, 100.0, 50.0), seed=3, m=50, k=10, t=2, s=120, tol=1e-7, sketch="sparse_sign",
               max_restarts=100),
    "c2": dict(n=128, beta=(100.0, 50.0, 25.0), seed=1, m=100, k=20, t=2, s=240, tol=1e-8, sketch="srdct",
               max_restarts=10),
}
METRIC = "gmres_sdr_arnoldi_steps_per_s"


def workload_config(name, wl, world):
    """The `config` both arms print (identical dicts): the workload — the
    global problem (7-point convection-diffusion on n^3, Dirichlet: 7 n^3 -
    6 n^2 stored entries), the solver parameters, the row partition. How a
    rank stores its block is an implementation detail (`storage`, top level)."""
    n = wl["n"]
    N = n ** 3
    return {"workload": name, "N": N, "N_per_gpu": N // world, "nnz": 7 * n ** 3 - 6 * n ** 2, "m": wl["m"],
            "k": wl["k"], "t": wl["t"], "s": wl["s"], "tol": wl["tol"], "max_restarts": wl["max_restarts"],
            "sketch": wl["sketch"], "parallelism": f"zslab{world}",
            "l2": "inputs larger than L2 (Krylov basis (m+1) x 8N bytes per cycle, no L2 flush)"}
STEP_KERNELS = ("spmv_arnoldi", "update", "sketch", "update_sketch", "sketch_fold", "fold_partials")
# one GPU, sparse sign: KF does the update of step j and the SpMV of step j+1
# in one launch; a cycle's first SpMV (K1) and last update (K2s), and the
# w_0 = r0 pass, are the other step launches
FUSED_STEP_KERNELS = ("fused_step", "fused_fold", "spmv_arnoldi", "update_sketch", "sketch_fold")


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_info():
    """CPU model, logical cores and RAM of the box the CPU baseline runs on."""
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                ram = round(int(ln.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gib": ram}


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed
    region through NVML (the library nvidia-smi queries)."""

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
    """B_step = bytes(A) + 8 N (4 + 2t); bytes(A) = the
    operator storage one SpMV streams (`A.storage["bytes"]`: SELL-DIA 8 B per
    stored entry here; the reference's CSR 12 nnz + 4 (N + 1) for §8(d)'s figure)."""
    return a_bytes + 8 * N * (4 + 2 * t)


def kernel_bytes(N, a_bytes, t, sketch):
    """Algorithmic bytes per launch of each step kernel."""
    return {
        "spmv_arnoldi": a_bytes + 8 * N * (2 + (t - 1)),          # A, x read, y written, t-1 window reads
        "update": 8 * N * (1 + t) + 8 * N,                        # y + t window reads, w written
        "update_sketch": 8 * N * (1 + t) + 8 * N + (N // 8 if sketch == "srdct" else 0),  # fused: + sign bits
        "sketch": 8 * N + (N // 8 if sketch == "srdct" else 0),  # one read of w (+ sign bits)
        # KF: A, y_j and the t window columns read, w_{j+1} and y_{j+1} written
        # (the SpMV's reads of w_{j+1} and w_j come back from L2)
        "fused_step": a_bytes + 8 * N * (1 + t) + 8 * N * 2,
    }


def oracle_sample(wl, steps, all_cores=False):
    """The CPU oracle on the workload: builds A (direct CSR), b and the sketch,
    runs init_krylov once and `steps` solve_cycle steps; per-step seconds.
    all_cores: then the same sample again with the oracle's long loops split
    over every host core (ORC_THREADS; the reference itself is single-threaded)."""
    from oracle import pyoracle as O
    n = wl["n"]
    N = n ** 3
    t0 = time.time()
    A = O.gen_convdiff3d(n, *wl["beta"])
    b = O.gaussian_vector(N, wl["seed"])
    S = (O.SketchOperator.subsampled_dct(N, wl["s"], 0x5EED) if wl["sketch"] == "srdct"
         else O.SketchOperator.sparse_sign(N, wl["s"], 0x5EED, 8))
    setup = time.time() - t0
    done, init_s, step_s = O.step_sample(A, b, S, wl["t"], steps)
    assert done == steps, (done, steps)
    out = dict(N=N, nnz=A.nnz, setup_s=setup, init_s=init_s, step_s=step_s, steps=steps)
    if all_cores:
        nt = os.cpu_count() or 1
        old = os.environ.get("ORC_THREADS")
        os.environ["ORC_THREADS"] = str(nt)
        try:
            done, _, step_mt = O.step_sample(A, b, S, wl["t"], steps)
        finally:
            if old is None:
                os.environ.pop("ORC_THREADS", None)
            else:
                os.environ["ORC_THREADS"] = old
        out.update(step_s_all_cores=step_mt, threads=nt)
    return out


def run_reference(args, wl, rank, world):
    """--impl reference: the CPU oracle on the same workload (rank 0 only)."""
    if rank != 0:
        return None
    warm = min(args.warmup, 1)
    # steps are timed as a whole after one warm step (the per-step work is identical)
    from oracle import pyoracle as O  # noqa: F401
    r = oracle_sample(wl, warm + args.steps, all_cores=True)
    # the reference arm runs with every host thread it can use: the oracle's
    # long loops (SpMV, vector passes, sparse sign) split over all cores
    # (the faster of the all-threads and the one-thread run: the SRDCT
    # workloads are DCT-bound and the DCT is not split, so threads can lose)
    one_thread = r["steps"] / r["step_s"]
    threads = r["threads"] if r["step_s_all_cores"] < r["step_s"] else 1
    per_step = min(r["step_s_all_cores"], r["step_s"]) / r["steps"]
    value = 1.0 / per_step
    sample = (f"{args.config} at full size (N={r['N']}): init_krylov once ({r['init_s']:.1f} s, untimed), then "
              f"{warm}+{args.steps} solve_cycle steps (arnoldi_step + IncrementalQR append + LS solve, "
              f"solver.hpp:165-179), 1 step per bench step; oracle C++ restatement (the reference is unbuildable "
              f"here), the faster of {r['threads']} host threads ({r['steps'] / r['step_s_all_cores']:.3f} steps/s) "
              f"and 1 thread ({one_thread:.3f} steps/s; the reference itself is single-threaded)")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generators, seeded)",
        "config": workload_config(args.config, wl, world),
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": threads, "kind": "port", "sample": sample,
                         "one_thread": {"value": one_thread, "unit": "steps/s"}, **host_info()},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": r["setup_s"],
    }


_JSON_OUT = None


def emit(line):
    """The one JSON line on the real stdout (library / NCCL banners that write to
    fd 1 during the run are sent to stderr, see __main__)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def relaunch(ngpus):
    """bench.py --gpus N outside torchrun: N ranks through torch.distributed.run
    on this node (127.0.0.1), NCCL_DEBUG=INFO so the communicator set-up is logged."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    wl = WORKLOADS[args.config]
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE {world}; using {world} ranks", file=sys.stderr)

    if args.impl == "reference":
        line = run_reference(args, wl, rank, world)
        if line is not None:
            emit(line)
        return

    # SDR_BENCH_HOSTCOMM=1: the ranks share GPU 0 and exchange through the
    # host-staged transport (gloo) instead of NCCL — a one-GPU check of the
    # multi-rank bench logic (slabs, max over ranks, e2e), not a measurement
    hostcomm = os.environ.get("SDR_BENCH_HOSTCOMM") == "1" and world > 1
    if hostcomm:
        local = 0
    import torch
    torch.cuda.set_device(local)
    import paper_2311_14206_b200 as sk

    # SDR_BENCH_DIST=1 takes the multi-GPU code path even on one rank (one-rank
    # NCCL communicator): a check of the torchrun / NCCL plumbing on one GPU
    if world > 1 or os.environ.get("SDR_BENCH_DIST") == "1":
        import torch.distributed as dist
        if "RANK" not in os.environ:  # SDR_BENCH_DIST=1 without a launcher: a one-rank group
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1")
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(so.getsockname()[1])
        dist.init_process_group("gloo", init_method="env://")
        if hostcomm:
            ctx = sk.Context(local, rank, world, host_comm=sk.torch_host_comm())
        else:
            idbuf = [sk.Context.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(idbuf, src=0)
            ctx = sk.Context(local, rank, world, idbuf[0])
    else:
        dist = None
        ctx = sk.Context(local)

    n = wl["n"]
    z0, z1 = n * rank // world, n * (rank + 1) // world  # z-slab of the global grid (strong scaling)
    t_setup = time.time()
    A = sk.SparseMatrix.convdiff3d_device(n, *wl["beta"], z_begin=z0, z_end=z1, ctx=ctx)
    N = A.rows
    nloc = A.local_rows
    # b = gaussian_vector(N, seed): every rank draws the same stream and keeps its block
    b_full = sk.gaussian_vector(N, wl["seed"])
    b_host = torch.from_numpy(np.ascontiguousarray(b_full[A.row_begin:A.row_begin + nloc])).pin_memory()
    del b_full
    b_dev = b_host.to(f"cuda:{local}")
    S = (sk.SketchOperator.subsampled_dct(N, wl["s"], 0x5EED, ctx=ctx) if wl["sketch"] == "srdct"
         else sk.SketchOperator.sparse_sign(N, wl["s"], 0x5EED, 8, ctx=ctx))
    cfg = sk.SolverConfig(m=wl["m"], k=wl["k"], t=wl["t"], s=wl["s"], tol=wl["tol"], max_restarts=wl["max_restarts"])
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
    setup_s = time.time() - t_setup

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, t)
        return max(float(g[0]) for g in gathered)

    def one(b, out=None):
        return sk.solve(A, b, cfg, space=sk.RecycleSpace(ctx), sketch=S, out=out)

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
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    # strong scaling: every rank takes the same (global) Arnoldi steps on its
    # slab; whole-job throughput = global steps / max-over-ranks time
    value = iters / (ms / 1e3)

    # ---- e2e through the public API with host buffers: H2D of b (pinned), D2H of x (pinned)
    x_host = torch.empty(nloc, dtype=torch.float64).pin_memory()
    one(b_host.numpy(), out=x_host.numpy())  # first-touch staging of the host-buffer path
    ctx.synchronize()
    barrier()
    e2e_iters = 0
    e2e_walls = []
    t_e2e0 = time.perf_counter()
    for _ in range(args.steps):
        tw = time.perf_counter()
        r = one(b_host.numpy(), out=x_host.numpy())
        e2e_iters += r.report.iterations
        e2e_walls.append(1e3 * (time.perf_counter() - tw))
    ctx.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t_e2e0)
    e2e_value = e2e_iters / e2e_s

    # ---- per-kernel in-solve durations: CUDA events around every launch of one
    # instrumented solve (on the library stream)
    ctx.set_timing(True)
    ctx.timing_reset()
    rt = one(b_dev)
    ctx.synchronize()
    names = ("spmv_arnoldi", "update", "sketch", "update_sketch", "sketch_fold", "sketch_side", "tallskinny",
             "recycle_gemm", "col_norms", "correction", "residual", "copy_norm", "allreduce", "halo", "axpy",
             "fold_partials", "fused_step", "fused_fold")
    ktimes = {k: ctx.timing(k) for k in names}
    ctx.set_timing(False)
    kb = kernel_bytes(nloc, A.storage["bytes"], wl["t"], wl["sketch"])
    peak, peak_kind = measured_peak()
    kern = {}
    for name, (cnt, tot) in ktimes.items():
        if cnt:
            d = {"launches": cnt, "avg_us": 1e3 * tot / cnt, "share": 0.0}
            if name in kb:
                d["bytes"] = kb[name]
                d["GBps"] = kb[name] / (tot / cnt * 1e-3) / 1e9
                d["frac"] = d["GBps"] / peak
            kern[name] = d
    tot_all = sum(v["avg_us"] * v["launches"] for v in kern.values())
    for v in kern.values():
        v["share"] = v["avg_us"] * v["launches"] / tot_all if tot_all else 0.0
    dom = max((k for k in kern if k in kb), key=lambda k: kern[k]["avg_us"] * kern[k]["launches"])
    # the per-step kernels' time per Arnoldi step (a cycle's init sketch and
    # other once-per-cycle launches of the same names are left out)
    its = rt.report.iterations
    if "fused_step" in kern:
        # every launch of the step kernels, a cycle's w_0 = r0 pass and the
        # speculative steps past a trigger included (conservative)
        per_step = [k for k in FUSED_STEP_KERNELS if k in kern]
    else:
        per_step = [k for k in STEP_KERNELS if k in kern and kern[k]["launches"] >= its]
    step_us = sum(kern[k]["avg_us"] * kern[k]["launches"] for k in per_step) / max(1, its)
    step_bytes = bytes_per_step(nloc, A.storage["bytes"], wl["t"])
    csr_bytes = bytes_per_step(nloc, 12 * A.nnz + 4 * (nloc + 1), wl["t"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as fh:
            traffic = json.load(fh).get(args.config, {}).get(dom)
    except Exception:
        pass
    dom_us = kern[dom]["avg_us"]
    dom_gbps = kb[dom] / (dom_us * 1e-6) / 1e9
    solve_ms = ms / args.steps
    per_step_all_us = 1e3 * solve_ms / max(1, iters // args.steps)
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": dom_gbps, "peak": peak, "unit": "GB/s", "frac": dom_gbps / peak,
        "traffic": traffic, "peak_source": peak_kind, "bytes_per_launch": kb[dom], "launch_us": dom_us,
        "method": "CUDA events around every launch of one instrumented solve (library stream); algorithmic bytes "
                  "per launch from the operator's storage (DESIGN.md §4)",
        "arnoldi_step": {"bytes": step_bytes, "us": step_us, "GBps": step_bytes / (step_us * 1e-6) / 1e9,
                         "frac": step_bytes / (step_us * 1e-6) / 1e9 / peak,
                         "kernels": per_step,
                         "timer": "in-solve launch durations of the per-step kernels, summed per Arnoldi step"},
        "whole_solve_per_step": {"bytes_storage": step_bytes, "bytes_csr_8d": csr_bytes, "us": per_step_all_us,
                                 "frac_storage": step_bytes / (per_step_all_us * 1e-6) / 1e9 / peak,
                                 "frac_csr_8d": csr_bytes / (per_step_all_us * 1e-6) / 1e9 / peak,
                                 "timer": "timed solve / Arnoldi steps (restarts, verifications and recycle "
                                          "updates included)"},
    }

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_sample(wl, 2, all_cores=True)
        v = r["steps"] / r["step_s"]
        cpu_baseline = {"value": v, "unit": "steps/s", "cores": 1, "kind": "port",
                        "sample": (f"{args.config} at full size (N={r['N']}): init_krylov ({r['init_s']:.1f} s, "
                                   f"untimed) then {r['steps']} solve_cycle steps (arnoldi_step + QR append + LS "
                                   f"solve), oracle C++ restatement on 1 host thread (the reference is "
                                   f"single-threaded); {r['step_s']:.1f} s of CPU work"),
                        "time_to_solution_s_extrapolated": rt.report.iterations / v,
                        "all_cores": {"value": r["steps"] / r["step_s_all_cores"], "unit": "steps/s",
                                      "threads": r["threads"],
                                      "note": "the oracle's SpMV, vector and sparse-sign loops over every host "
                                              "core (a secondary figure; the reference is single-threaded)"},
                        **host_info()}

    if rank == 0:
        rep = reports[-1]
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": solve_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE generators, seeded)",
            "config": workload_config(args.config, wl, world),
            "storage": dict(A.storage, rank0_rows=nloc, rank0_nnz=A.nnz),
            **({"transport": "host-staged test transport (SDR_BENCH_HOSTCOMM, ranks share GPU 0)"} if hostcomm else {}),
            "time_to_solution_ms": solve_ms,
            "solve": {"status": rep.status, "iterations": rep.iterations, "cycles": rep.cycles,
                      "final_relative_residual": rep.final_relative_residual,
                      "wall_ms": [round(v, 1) for v in walls], "e2e_wall_ms": [round(v, 1) for v in e2e_walls],
                      "phases_ms": {k: round(v, 1) for k, v in rep.phases.items()}},
            "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": 8 * nloc,
                    "d2h_bytes_per_step": 8 * nloc,
                    "path": "sdr_solve with host (pinned) b and host x, copies inside the timed region"},
            "roofline": roofline,
            "kernels": kern,
            "cpu_baseline": cpu_baseline,
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "setup_s": round(setup_s, 2),
        }
        emit(line)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    _ngpus = 1
    for _i, _a in enumerate(sys.argv):
        if _a == "--gpus" and _i + 1 < len(sys.argv):
            _ngpus = int(sys.argv[_i + 1])
        elif _a.startswith("--gpus="):
            _ngpus = int(_a.split("=", 1)[1])
    if _ngpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(_ngpus))
    if (os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION" and "SDR_BENCH_REEXEC" not in os.environ
            and "reference" not in sys.argv and "--impl=reference" not in sys.argv):
        # the communicator set-up lines (NCCL_DEBUG=INFO) for the log; NCCL
        # takes its debug level from the environment the process starts
        # with, so re-exec once with it (an interpreter start-up hook on the
        # GPU boxes presets VERSION, which prints the version banner only)
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["SDR_BENCH_REEXEC"] = "1"
        sys.stdout.flush()
        os.execv(sys.executable, [sys.executable] + sys.argv)
    # keep stdout for the JSON line alone: fd 1 points at stderr while the
    # workload runs (NCCL prints its version banner to stdout on rank 0)
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    main()
