"""bench.py's JSON contract on the CPU: the reference arm (the oracle port,
whole frames) on config 1 prints one line with the keys the driver reads."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    env = dict(os.environ, SFB_REF_BUDGET_S="30")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config",
                          "c1", "--steps", "2", "--warmup", "0"],
                         capture_output=True, text=True, check=True, env=env, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert 1 <= d["steps_sampled"] <= 2
    assert "extrapolat" not in d["cpu_baseline"]["sample"]   # whole frames only
