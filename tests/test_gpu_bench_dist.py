"""bench.py under torchrun with two ranks (the driver's
SCALE launch): the ranks share GPU 0 through the host-staged transport
(SDR_BENCH_HOSTCOMM=1), so the multi-rank bench logic — z-slabs of the
global grid, strong-scaled steps/s, max over ranks, e2e with per-rank host
buffers — and the solver's rank-invariant collective order (lockstep step
issue, solver.cpp ArnoldiPipeline::lockstep) run end to end. C2 on two slabs
must take the single-GPU solve's 380 iterations (tests/golden C2)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_c2_strong_scaled():
    env = dict(os.environ, SDR_BENCH_HOSTCOMM="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--config", "c2", "--steps", "2",
           "--warmup", "1"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["parallelism"] == "zslab2" and d["config"]["N_per_gpu"] * 2 == d["config"]["N"]
    assert d["solve"]["status"] == "converged" and d["solve"]["iterations"] == 380
    assert d["solve"]["final_relative_residual"] < 1e-8
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
