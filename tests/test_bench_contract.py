"""bench.py's reference arm (the oracle on the host, no GPU) prints the contract's JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_json_line():
    d = run_bench("--impl", "reference", "--config", "cfg0", "--steps", "2", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["cpu_baseline"]["nproc"] >= 1 and "pinned_core" in d["cpu_baseline"]
    assert d["config"]["workload"] == "cfg0" and d["dtype"] == "f64"


def test_reference_arm_warmup_floor():
    d = run_bench("--impl", "reference", "--config", "cfg0", "--steps", "1", "--warmup", "0")
    assert d["warmup"] == 3                   # W >= 3 is enforced
