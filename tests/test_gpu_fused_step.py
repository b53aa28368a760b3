"""KF, the opt-in one-launch Arnoldi step (fused_step.cu, SDR_FUSE_STEP=1):
its parity cases (tests/workers/fused_step_cases.py — H, SV, SAV, V within
1e-12 of the oracle's truncated Arnoldi, chunk waits, long stencil reach,
ragged lengths, bitwise reproducibility, a C5-parameter solve) in a
subprocess, since the switch is read once per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fused_step_opt_in_path_matches_oracle():
    env = dict(os.environ, SDR_FUSE_STEP="1")
    cmd = [sys.executable, "-m", "pytest", "tests/workers/fused_step_cases.py", "-q", "-x", "-p", "no:cacheprovider"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
