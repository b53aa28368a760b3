"""The C-ABI from plain C++ (examples/solve_c2.cpp, no Python in the
process): build it, run a C2-shaped solve with host b / x and a second
right-hand side on the carried recycle space, check the residual verified
through the device SpMV."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cxx_caller_solves(sk):
    subprocess.run(["make", "-s", "examples"], cwd=ROOT, check=True, capture_output=True, timeout=300)
    p = subprocess.run([os.path.join(ROOT, "examples", "solve_c2"), "48"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("system")]
    assert len(lines) == 2 and all("status 0" in ln for ln in lines)
    for ln in lines:  # the host-side verified residual meets the tolerance
        verified = float(ln.split("verified ")[1].split(")")[0])
        assert verified <= 1e-8 * 1.01
