"""Full size, full step count: every BASELINE.json configuration at its own grid size over its whole horizon
(Algorithm 1's time loop) on the GPU, in the bench's launch configuration (CUDA-graph
batches), against the oracle's result of the same run stored by tools/oracle_digests.py (which calls only
oracle/ and workloads/): tests/golden/full_size_digests.json (SHA-256 of the final float64 rasters, of the dt
sequence and of the packed wet mask) and tests/golden/full_size/<cfg>.npz (the whole dt sequence and the
final state at 4096 seeded sample cells).

North_star tolerances: max |dh|, |dhu|, |dhv| (and |dV|) <= 1e-8 after the full count -- checked on the
samples --, the wet/dry mask identical (its digest), the dt sequence equal to 1e-13 relative, the same step
count and final time; and, the kernels being bit-identical to the oracle (DESIGN.md §3 "contract"), equal
digests: every cell of every field and every dt equal bit for bit.
A configuration whose digest was not generated yet is skipped with that reason; a digest whose oracle or
workload sources changed since it was written fails (it would no longer describe this oracle).
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from swof_testlib import gpu_solver
from workloads import make

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"
TOL_FULL = 1e-8


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _source_digest():
    h = hashlib.sha256()
    for p in ("oracle/swof_oracle.c", "oracle/swof_oracle.h", "workloads/configs.py", "workloads/rng.py",
              "workloads/dem.py"):
        h.update((ROOT / p).read_bytes())
    return h.hexdigest()


def _entry(name):
    data = json.loads((GOLD / "full_size_digests.json").read_text())
    ent = data.get(name)
    npz = GOLD / "full_size" / f"{name}.npz"
    if ent is None or not npz.exists():
        pytest.skip(f"{name}: full-size oracle result not generated yet (tools/oracle_digests.py {name})")
    assert ent["source_sha"] == _source_digest(), f"{name}: digest is stale (oracle/workload sources changed)"
    return ent, np.load(npz)


def _make(name):
    """'cfgK': full size, full count; 'cfgK@N': the same full-size inputs over the first N steps (for the
    configurations whose full count takes the oracle hours on the host: cfg3, cfg4)."""
    base, _, n = name.partition("@")
    cfg = make(base)
    if n:
        cfg.steps = int(n)
    return cfg


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg3@500", "cfg3@1000", "cfg3@2000", "cfg4@100", "cfg4@300"])
def test_full_size_full_count(gpu, name):
    ent, ref = _entry(name)
    cfg = _make(name)
    assert (cfg.nx, cfg.ny) == (ent["nx"], ent["ny"])
    s = gpu_solver(cfg, graph_steps=16)
    if cfg.t_end is not None:
        s.run(cfg.t_end, 1 << 40)
    else:
        s.step(cfg.steps)
    g = s.get_state()
    dt = s.dt_history()
    d = s.diag()
    s.close()
    assert d["flags"] == 0
    assert g["step"] == ent["steps"] and len(dt) == len(ref["dt"])
    assert abs(g["t"] - ent["t"]) <= 1e-13 * ent["t"]
    assert np.max(np.abs(dt / ref["dt"] - 1.0)) <= 1e-13
    # the wet/dry mask, cell for cell
    mask = hashlib.sha256(np.packbits(np.ascontiguousarray(g["h"] > cfg.h_eps)).tobytes()).hexdigest()
    assert mask == ent["sha_mask"] and int(np.count_nonzero(g["h"] > cfg.h_eps)) == ent["wet"]
    idx = ref["idx"]
    keys = ["h", "hu", "hv"] + (["v"] if cfg.ga is not None else [])
    worst = {k: float(np.max(np.abs(g[k].ravel()[idx] - ref[k]))) for k in keys}
    for k in keys:
        assert worst[k] <= TOL_FULL, (k, worst[k])
    bitwise = (_sha(g["h"]) == ent["sha_h"] and _sha(g["hu"]) == ent["sha_hu"] and _sha(g["hv"]) == ent["sha_hv"]
               and (cfg.ga is None or _sha(g["v"]) == ent["sha_v"]) and _sha(dt) == ent["sha_dt"])
    print(name, g["step"], "steps, sampled worst", worst, "bitwise (every cell, digests)", bitwise)
    assert bitwise
