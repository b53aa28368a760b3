"""The reference arm of bench.py (`--impl reference`) on CPU: the driver's JSON
contract — one line with impl, metric, unit, value, the workload config both
arms share, cpu_baseline (kind, cores, sample, host) and an e2e object with
no host-device bytes. C2 at full size, one timed step (about 10 s of CPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    sys.path.insert(0, ROOT)
    import bench

    cmd = [sys.executable, "bench.py", "--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "1"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC and d["unit"] == "steps/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 1
    assert d["config"] == bench.workload_config("c2", bench.WORKLOADS["c2"], 1)
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert cb["nproc"] >= cb["cores"] and cb["sample"] and cb["one_thread"]["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
