"""World-size-2 run of the PRODUCT's distributed pipeline on one GPU.

Two processes, one z-slab (or row block) each, run sdr_solve through the
distributed code path — halo plan and exchange, the K1 interior / boundary
split around the halo (per-row stencil reach), per-rank fixed-order folds of
the CTA partials, one reduced payload per Arnoldi step, replicated host QR /
harmonic restarts — with the host-staged transport (sdr_ctx_create_hostcomm,
gloo underneath). NCCL cannot put two ranks on one GPU, and ranks whose
kernels wait on one another must not share a GPU (B200_PROFILING.md), so
every collective here completes on the host between kernels.
The result must equal the one-rank solve: same status, iterations within
±2 %, x within 1e-9 relative."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.workers.dist_cases import CASES, build

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("case", sorted(CASES))
def test_two_ranks_match_one_rank(sk, tmp_path, case):
    out = str(tmp_path / case)
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK="0")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "workers", "dist_hostcomm_worker.py"),
                                       case, out], env=env, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        logs.append(o.decode(errors="replace"))
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)[-4000:]
    parts = [np.load(f"{out}.rank{r}.npz") for r in range(2)]

    A, b, S, cfg = build(sk, CASES[case], sk.default_context(), 0, 1)
    ref = sk.solve(A, b, cfg, sketch=S)
    x = np.concatenate([p["x"] for p in parts])
    it = int(parts[0]["iterations"])
    assert all(int(p["iterations"]) == it for p in parts)  # replicated host state: every rank takes the same steps
    assert str(parts[0]["status"]) == ref.report.status == "converged"
    assert abs(it - ref.report.iterations) <= max(1, 0.02 * ref.report.iterations), (it, ref.report.iterations)
    assert float(parts[0]["final"]) < CASES[case]["tol"]
    assert np.linalg.norm(x - ref.x) <= 1e-9 * np.linalg.norm(ref.x), np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)
