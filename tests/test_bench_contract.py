"""bench.py contract on CPU: the reference arm (the unmodified reference on host cores, or the
oracle port when it is not installed) prints ONE JSON line with the driver's keys.  The GPU arm's
line is exercised by the driver on a B200."""

import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-sample", "16"],
        capture_output=True, text=True, timeout=300, cwd=ROOT, env={**os.environ, "RANK": "0", "WORLD_SIZE": "1"},
    )
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "cfg2"
    from oracle import reference_arm as R

    assert d["cpu_baseline"]["kind"] == ("reference" if R.locate() else "port") and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_nonzero_rank_is_silent():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-sample", "16"],
        capture_output=True, text=True, timeout=300, cwd=ROOT, env={**os.environ, "RANK": "1", "WORLD_SIZE": "2"},
    )
    assert out.returncode == 0 and out.stdout.strip() == ""
