"""Full-size, full-step-count oracle results of BASELINE.json's configurations, stored as digests.

Writes tests/golden/full_size_digests.json (calls only oracle/ and workloads/; no value comes from the CUDA
path).  For each configuration at its full size the oracle (the OpenMP-over-rows build, bitwise identical to
the serial one: tests/test_oracle_omp.py) runs the configuration's whole horizon (Algorithm 1's time loop,
PAPER.md P:773-788) and the file records SHA-256 digests of the final h, hu, hv, V rasters (float64, row-major)
and of the dt sequence, the SHA-256 of the packed wet mask (h > h_eps), plus summary values for diagnosis;
tests/golden/full_size/<cfg>.npz holds the whole dt sequence and the final h, hu, hv, V at 4096 seeded sample
cells (so that a GPU build that is not bitwise can still be held to the north_star tolerances: <= 1e-8 on the
samples, the identical wet mask by its digest, dt to 1e-13).  tests/test_gpu_full_size.py runs the GPU path on
the same inputs and compares digests: equal digests mean the GPU state equals the oracle's bit for bit
(hence within every north_star tolerance, masks and dt sequence included).

    OMP_NUM_THREADS=7 python tools/oracle_digests.py cfg1 cfg2 cfg4 cfg3
    OMP_NUM_THREADS=7 python tools/oracle_digests.py cfg4@100 cfg3@500     # full size, the first N steps
    python tools/oracle_digests.py cfg3 --ckpt /tmp/swof_ckpt --max-seconds 3000   # resumable, in chunks

With --ckpt the run advances in chunks of 50 steps and, when --max-seconds is spent, saves the state (h, hu, hv,
V, t), the dt sequence so far and the clamp counters to DIR/<cfg>.npz and exits with status 3; the next call
resumes from it.  Chunked and unchunked runs give the same state bit for bit (each step is a function of the
state only; the chunk boundary passes the state through unchanged).

Run time on 8 host cores: cfg1 ~7 min, cfg2 ~15 min, cfg4 ~4 h, cfg3 ~5 h (cfg4 needs ~36 GB of RAM).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from workloads import make  # noqa: E402

OUT = ROOT / "tests" / "golden" / "full_size_digests.json"
NPZ = ROOT / "tests" / "golden" / "full_size"
N_SAMPLES = 4096


def make_named(name: str):
    """'cfgK' = configuration K at full size over its whole horizon; 'cfgK@N' = the same full-size inputs
    over the first N steps only (a step-count configuration's prefix: cfg3, cfg4)."""
    base, _, n = name.partition("@")
    cfg = make(base)
    if n:
        assert cfg.steps is not None and cfg.t_end is None, f"{base} is not a step-count configuration"
        cfg.steps = int(n)
    return cfg


def sample_index(name: str, ncell: int) -> np.ndarray:
    """The sampled cells (flat row-major indices): a seeded draw, sorted, plus the first and last cell."""
    rs = np.random.default_rng(int.from_bytes(hashlib.sha256(name.encode()).digest()[:8], "little"))
    return np.unique(np.concatenate([[0, ncell - 1], rs.integers(0, ncell, N_SAMPLES - 2)]))


def mask_sha(h, h_eps) -> str:
    return hashlib.sha256(np.packbits(np.ascontiguousarray(h > h_eps)).tobytes()).hexdigest()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def source_digest() -> str:
    """The oracle's arithmetic and the input generator: digests are stale if either changes."""
    h = hashlib.sha256()
    for p in ("oracle/swof_oracle.c", "oracle/swof_oracle.h", "workloads/configs.py", "workloads/rng.py",
              "workloads/dem.py"):
        h.update((ROOT / p).read_bytes())
    return h.hexdigest()


class _Cnt:
    def __init__(self, clamps, clamp_max):
        self.clamps, self.clamp_max = clamps, clamp_max


def run_chunked(cfg, name, ckpt, max_seconds, t0, chunk=50):
    """Advance cfg's full horizon in chunks of `chunk` steps from DIR/<name>.npz (if present); returns
    (result dict, elapsed oracle seconds incl. earlier calls) when done, or (None, _) after checkpointing."""
    path = Path(ckpt) / f"{name}.npz"
    total = cfg.steps if cfg.steps is not None else 1 << 40
    t_end = cfg.t_end if cfg.t_end is not None else float("inf")
    if path.exists():
        c = np.load(path)
        h, hu, hv = c["h"], c["hu"], c["hv"]
        v = c["v"] if c["v"].size else None
        t, dts, clamps, cmax, spent = float(c["t"]), list(c["dt"]), int(c["clamps"]), float(c["cmax"]), float(c["spent"])
    else:
        h, hu, hv = cfg.h, cfg.hu, cfg.hv
        v = cfg.vinf if cfg.ga is not None else None
        t, dts, clamps, cmax, spent = 0.0, [], 0, 0.0, 0.0
    while len(dts) < total and t < t_end:
        r = oracle.run(cfg, h=h, hu=hu, hv=hv, v=v, t0=t, nsteps=min(chunk, total - len(dts)), omp=True)
        assert r["rc"] == 0, r["rc"]
        h, hu, hv, v, t = r["h"], r["hu"], r["hv"], r["v"], r["t"]
        dts.extend(r["dt"].tolist())
        clamps += int(r["counters"].clamps)
        cmax = max(cmax, float(r["counters"].clamp_max))
        if r["steps"] == 0:
            break
        if len(dts) % 500 == 0:
            print(f"{name}: {len(dts)} steps, t = {t:.6g}, {spent + time.time() - t0:.0f} s", file=sys.stderr, flush=True)
        if time.time() - t0 > max_seconds and len(dts) < total and t < t_end:
            Path(ckpt).mkdir(parents=True, exist_ok=True)
            np.savez(path, h=h, hu=hu, hv=hv, v=(v if v is not None else np.zeros(0)), t=t, dt=np.array(dts),
                     clamps=clamps, cmax=cmax, spent=spent + time.time() - t0)
            return None, None
    res = {"rc": 0, "h": h, "hu": hu, "hv": hv, "v": v, "t": t, "steps": len(dts), "dt": np.array(dts),
           "counters": _Cnt(clamps, cmax)}
    return res, spent + time.time() - t0


def main(names, ckpt=None, max_seconds=float("inf")):
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    data["_source"] = ("tools/oracle_digests.py: oracle (OpenMP-over-rows build, bitwise = serial) at each "
                       "configuration's full size and full step count; SHA-256 of the float64 rasters")
    src = source_digest()
    for name in names:
        cfg = make_named(name)
        t0 = time.time()
        if ckpt is None:
            r = oracle.run(cfg, omp=True)
            el = time.time() - t0
            assert r["rc"] == 0, r["rc"]
        else:
            r, el = run_chunked(cfg, name, ckpt, max_seconds, t0)
            if r is None:
                print(name, "checkpointed", flush=True)
                sys.exit(3)
        h = r["h"]
        ent = {
            "nx": cfg.nx, "ny": cfg.ny, "steps": int(r["steps"]), "t": r["t"], "t_end": cfg.t_end,
            "sha_h": sha(h), "sha_hu": sha(r["hu"]), "sha_hv": sha(r["hv"]),
            "sha_v": sha(r["v"]) if r["v"] is not None else None,
            "sha_dt": sha(r["dt"]), "dt_first": float(r["dt"][0]), "dt_last": float(r["dt"][-1]),
            "sha_mask": mask_sha(h, cfg.h_eps), "wet": int(np.count_nonzero(h > cfg.h_eps)), "sum_h": float(oracle.pairwise_sum(h)),
            "max_h": float(h.max()), "clamps": int(r["counters"].clamps),
            "clamp_max": float(r["counters"].clamp_max), "source_sha": src,
            "oracle_seconds": round(el, 1), "threads": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())),
        }
        idx = sample_index(name, h.size)
        NPZ.mkdir(parents=True, exist_ok=True)
        np.savez_compressed(NPZ / f"{name}.npz", idx=idx, dt=r["dt"], h=h.ravel()[idx], hu=r["hu"].ravel()[idx],
                            hv=r["hv"].ravel()[idx],
                            v=(r["v"].ravel()[idx] if r["v"] is not None else np.zeros(0)))
        data = json.loads(OUT.read_text()) if OUT.exists() else data  # other runs may have written meanwhile
        data[name] = ent
        OUT.write_text(json.dumps(data, indent=1) + "\n")
        print(name, json.dumps(ent), flush=True)


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["cfg1", "cfg2", "cfg4", "cfg3"])
    ap.add_argument("--ckpt", default=None)
    ap.add_argument("--max-seconds", type=float, default=float("inf"))
    a = ap.parse_args()
    main(a.names, a.ckpt, a.max_seconds)
