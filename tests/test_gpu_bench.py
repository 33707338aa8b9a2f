"""bench.py's own arm on the GPU prints the contract's JSON line (a small grid so it runs in seconds): the
metric, device and end-to-end values, the roofline object for the dominant kernel, the CPU oracle baseline,
the clocks sampled during the timed region and the launch count; and the D8 workload's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


def test_bench_json_line(gpu):
    d = run_bench("--nx", "512", "--ny", "384", "--steps", "4", "--warmup", "3", "--cpu-crop", "96",
                  "--cpu-steps", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline", "cpu_baseline"):
        assert k in d, k
    assert d["steps"] == 4 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0 and d["dtype"] == "f64"
    assert d["config"]["workload"] == "cfg4" and d["config"]["nx"] == 512 and d["config"]["ny"] == 384
    assert d["gpu_launches"] == 2 * d["steps"]
    e = d["e2e"]
    assert 0 < e["value"] < d["value"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "alu") and 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # the bound is the floor with the larger fraction; both floors and the step fractions are reported
    fl = r["floors"]
    assert r["frac"] == max(fl["hbm"]["frac"], fl["fp64"]["frac"])
    assert r["bound"] == ("hbm" if fl["hbm"]["frac"] >= fl["fp64"]["frac"] else "alu")
    st = r["step"]
    assert st["R_alg"] >= st["R_2k"] > 0 and abs(st["frac_R_alg"] - d["value"] / st["R_alg"]) < 1e-9
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] == 1 and c["value"] > 0 and "sample" in c
    assert c["nproc"] >= 1 and c["cpu_model"] and c["pinned_core"] >= 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_bench_d8_json_line(gpu):
    d = run_bench("--workload", "d8", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert d["value"] > 0 and d["unit"] == "points/s" and d["dtype"] == "f32"
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1
    assert d["vs_baseline"] is None and d["context"]["paper_seconds_per_pass"] == 31.0


def test_bench_shard_json_line(gpu):
    """The multi-GPU default (row strips; here one strip on one GPU through the same code path): the line
    carries the strong-scaling fields, the end-to-end value and the step-level roofline."""
    d = run_bench("--shard", "--nx", "512", "--ny", "384", "--steps", "4", "--warmup", "3")
    assert d["scaling"] == "strong" and d["n_gpus"] == 1 and d["value"] > 0 and d["step"] == 4
    assert 0 < d["e2e"]["value"] < d["value"] and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1
