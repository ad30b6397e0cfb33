"""CPU: bench.py's reference arm (the CPU oracle timed on host cores) keeps the JSON contract."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=300, env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout


def test_reference_arm_json():
    line = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1"])
    d = json.loads(line.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("tiny")


def test_reference_arm_nonzero_rank_exits_quietly():
    out = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "0",
                "--gpus", "2"], env={"RANK": "1", "WORLD_SIZE": "2"})
    assert out.strip() == ""
