"""CPU: bench.py's reference arm (the C oracle on host cores) prints one
JSON line with the contract's keys; nothing here needs a GPU."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--workload",
         "er2000", "--k", "4", "--steps", "2", "--warmup", "1", "--cpu-sample-s", "0.5"],
        capture_output=True, text=True, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"] == "er2000"


def test_b200_auto_rule():
    sys.path.insert(0, REPO)
    from paper_2104_13209_b200.cli import b200_auto

    assert b200_auto(4) == ("orient", "vertex")
    assert b200_auto(10) == ("pivot", "edge")
