"""CUDA-event throughput of the time step on every BASELINE.json configuration at full size (SURVEY.md §4
T6), plus the scheme variants on cfg4: one JSON line per case (cell-updates/s, ms per step, kernel split)."""
import json
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch  # noqa: E402

from paper_1307_4839_b200 import Solver, params_from_config  # noqa: E402
from workloads import make  # noqa: E402

torch.cuda.set_device(0)
CASES = [("cfg4", {"flux": "rusanov", "cfl": 0.25}, 50), ("cfg4", {"order": 1, "cfl": 1.0}, 50),
         ("cfg4", {"cfl_mode": "face"}, 50), ("cfg4", {"ga_form": "darcy"}, 50)] if "--variants" in sys.argv else [
         ("cfg0", {}, 200), ("cfg1", {}, 200), ("cfg2", {}, 100), ("cfg3", {}, 100), ("cfg3", {"dry_skip": 1}, 100),
         ("cfg4", {}, 50), ("cfg4", {"dry_skip": 1}, 50),
         ("cfg4", {"flux": "rusanov", "cfl": 0.25}, 50), ("cfg4", {"order": 1, "cfl": 1.0}, 50),
         ("cfg4", {"cfl_mode": "face"}, 50), ("cfg4", {"ga_form": "darcy"}, 50)]
for name, kw, steps in CASES:
    t0 = time.time()
    cfg = make(name)
    import os
    for k, v in kw.items():
        if k == "_env":
            os.environ[v] = "1"
        else:
            setattr(cfg, k, v)
    cfg.clamp_fail = 1.0 if kw and "dry_skip" not in kw else 0.0   # variants: report throughput even where the variant clamps (DESIGN Q23)
    stream = torch.cuda.Stream()
    s = Solver(params_from_config(cfg), cfg.z, cfg.fric_field, stream=stream)
    if "_env" in kw:
        del os.environ[kw["_env"]]
    s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
    s.step(5)
    if name in ("cfg2", "cfg3"):
        s.step(50)                      # let water enter the initially dry domains
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    s.step(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kp = s.step_profiled(min(steps, 10))
    d = s.diag()
    rate = cfg.nx * cfg.ny * steps / (ms / 1e3)
    roof = {}
    if not kw:
        # rooflines as bench.py computes them for cfg4: HBM (algorithmic bytes of the per-stage design) and
        # fp64 lanes (algorithmic ops per cell-update from the oracle's branch counters on a centre crop)
        import bench
        peaks, src = bench.load_peaks()
        bp, bc = bench.bytes_per_cell_update(cfg.ga is not None, cfg.fric_field is not None)
        crop = min(256, cfg.nx, cfg.ny)
        _, cnt, _, nst, _ = bench.cpu_sample(cfg, crop, 4)
        f_alg = bench.f_alg_from_counters(cnt, cfg, nst, crop * crop)
        peak_gops = 148 * 64 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e9
        roof = {"bytes_per_cell_update": bp + bc, "hbm_frac": (bp + bc) * rate / 1e9 / peaks["hbm_gbs"],
                "f_alg_per_cell_update": f_alg, "alu_frac": f_alg * rate / 1e9 / peak_gops, "peak_source": src}
    print(json.dumps({"case": name, "variant": kw, "nx": cfg.nx, "ny": cfg.ny, "steps": steps, "roofline": roof,
                      "cell_updates_per_s": cfg.nx * cfg.ny * steps / (ms / 1e3), "ms_per_step": ms / steps,
                      "kernel_ms_per_step": [x / min(steps, 10) for x in kp], "wet_cells": d["wet_cells"],
                      "launches_per_step": s.launches_per_step(), "setup_s": round(time.time() - t0, 1)}),
          flush=True)
    s.close()
