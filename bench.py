#!/usr/bin/env python
"""Benchmark: the FullSWOF_2D explicit time step (one Heun step = one "step") on cfg4 (8192 x 8192, the
BASELINE.json throughput/roofline configuration), fp64, 1 x B200 per rank.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg4]
    python bench.py --workload d8 [--steps K] [--warmup W] [--d8-dtype f32|f64]

N > 1 is launched by torchrun; the ONE cfg4 grid is cut into row strips, one per rank (the paper's MPI
decomposition P:731-760; strong scaling): per step two NCCL halo exchanges of 2 rows x 3 fields
with each neighbour and one all-reduce(max) of the 2 CFL words (--shard-fused: the kernels push the boundary
rows into the neighbours' CUDA-IPC-mapped ghost rows instead).  --replicas runs N independent full replicas
(weak scaling, no data-path collective) instead.  Timing: W untimed steps, then exactly K steps bracketed by
barrier + cuda synchronize, CUDA events on the context's stream, max over ranks.  The inputs (4.6 GB of
fields) are far larger than the 126 MB L2, so no flush is needed between steps.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/sec (fp64, 1xB200)"
UNIT = "cell-updates/s"

# Algorithmic fp64 operations of the canonical sheet, each add/sub/mul/div/sqrt/min/max/abs/
# cube-root = 1: per cell and stage, per face by HLL branch, per cell and step.
OPS_CELL_STAGE = 4 + 64 + 28 + 1          # primitives, MUSCL (2 axes), update (2 axes), rain
OPS_GA = 10
OPS_FRIC_WET = {"manning": 13, "strickler": 13, "darcy_weisbach": 12, "chezy": 12}
OPS_FIELD = 3                               # g*(n*n), dt*gc per cell with a per-cell coefficient field
OPS_FACE = {"dry": 15, "left": 39, "right": 39, "mid": 63}
OPS_STEP = 8 + 11                           # Heun (with V), CFL speeds + max
# algorithmic DRAM bytes per cell-update of the per-stage design: predictor reads
# h,hu,hv,z (+V, +n) and writes h,hu,hv (+V); corrector reads U* and z (+V*, +n), U^n (+V^n), writes U^{n+1} (+V)
def bytes_per_cell_update(ga: bool, field: bool):
    pred = 8 * (4 + ga + field) + 8 * (3 + ga)
    corr = 8 * (4 + ga + field) + 8 * (3 + ga) + 8 * (3 + ga)
    return pred, corr


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def reduce_max(x: float, world: int, device=None) -> float:
    """Max of a per-rank scalar over all ranks (identity on one rank)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(world: int, cells: int, steps: int, max_ms: float) -> float:
    """Whole-job cell-updates/s: every rank advanced its own replica by `steps` steps; the job took the
    slowest rank's time."""
    return world * cells * steps / (max_ms / 1e3)


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def cpu_sample(cfg, crop: int, steps: int):
    """The oracle, as it stands, on a crop x crop window of the workload: (cell-updates/s, counters, secs)."""
    import oracle
    from workloads.configs import SwofConfig
    j0 = (cfg.ny - crop) // 2
    i0 = (cfg.nx - crop) // 2
    sl = (slice(j0, j0 + crop), slice(i0, i0 + crop))
    sub = SwofConfig(**{**cfg.__dict__, "nx": crop, "ny": crop})
    for k in ("z", "h", "hu", "hv", "vinf", "fric_field"):
        a = getattr(cfg, k)
        setattr(sub, k, None if a is None else np.ascontiguousarray(a[sl]))
    sub.bc = {"W": "wall", "E": "wall", "S": "wall", "N": "wall"}
    sub.inflow = {}
    host = host_info()
    old = os.sched_getaffinity(0)
    core = max(old)                                   # pin the single-threaded oracle to one core
    os.sched_setaffinity(0, {core})
    try:
        t0 = time.perf_counter()
        r = oracle.run(sub, nsteps=steps, t_end=float("inf"))
        secs = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, old)
    host["pinned_core"] = core
    return crop * crop * r["steps"] / secs, r["counters"], secs, r["steps"], host


def f_alg_from_counters(cnt, cfg, steps, cells):
    """Algorithmic fp64 ops per cell-update from the oracle's branch counters."""
    ops = cnt.cell_stage * OPS_CELL_STAGE
    ops += cnt.face_dry * OPS_FACE["dry"] + cnt.face_left * OPS_FACE["left"]
    ops += cnt.face_right * OPS_FACE["right"] + cnt.face_mid * OPS_FACE["mid"]
    if cfg.ga is not None:
        ops += cnt.cell_stage * OPS_GA
    if cfg.fric_law != "none":
        ops += cnt.cell_wet_fric * OPS_FRIC_WET[cfg.fric_law]
        if cfg.fric_field is not None:
            ops += cnt.cell_wet_fric * OPS_FIELD
    ops += steps * cells * OPS_STEP
    return ops / (steps * cells)

def host_info():
    """CPU model, nproc and the core the oracle sample is pinned to (SURVEY.md §8d timing protocol)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def fp64_issue_ceiling(peak_gops):
    """The FP64-pipe ceiling of the kernels' own instruction mix: the pipe's lane-op rate over the executed fp64
    lane-instructions per cell-update (DMUL/DADD/DFMA/DSETP warp-instructions per cell x 32, predictor +
    corrector) from the committed ncu capture (profiles/ncu_latest.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_latest.json")) as f:
            prof = json.load(f)
        per_cell = 0.0
        for k in prof["kernels"].values():
            mix = k.get("opcode_mix_per_cell", {})
            per_cell += sum(mix.get(op, 0.0) for op in ("DMUL", "DADD", "DFMA", "DSETP", "DMNMX"))
        if per_cell <= 0:
            return None
        return {"value": peak_gops * 1e9 / (32 * per_cell), "unit": UNIT,
                "fp64_lane_instr_per_cell_update": 32 * per_cell,
                "source": f"profiles/ncu_latest.json: {prof['report']}"}
    except Exception:
        return None


def roofline(peaks, src, peak_gops, f_alg, dom, dom_ms, dom_bytes, cells, value, ga, field):
    """SURVEY.md §8d.  The dominant kernel against both of its floors -- HBM (algorithmic bytes / launch time
    vs the measured copy bandwidth) and the fp64 pipe (algorithmic ops, div/sqrt/cube root = 1, vs 148 x 64
    lanes x clock) -- `bound` being the one with the larger fraction; and the whole step against R_2k (the
    per-stage design's bytes) and R_alg (the step-fused minimum bytes; the headline of §8d)."""
    hbm = peaks["hbm_gbs"]
    hbm_ach = dom_bytes / (dom_ms / 1e3) / 1e9
    # dominant kernel's algorithmic fp64 ops: the per-stage half of the per-cell work, plus (corrector) the
    # per-step Heun + CFL ops
    ops_dom = (f_alg - OPS_STEP) / 2 + (OPS_STEP if dom == "corrector" else 0)
    fp_ach = ops_dom * cells / (dom_ms / 1e3) / 1e9
    frac_h, frac_f = hbm_ach / hbm, fp_ach / peak_gops
    traffic, tsrc, ncu = None, None, None
    try:   # DRAM read+write per launch of the same kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_latest.json")) as f:
            prof = json.load(f)
        for kname, k in prof["kernels"].items():
            is_corr = re.search(r"(stage|march)_kernel<(\(bool\))?(1|true)\b", kname) is not None
            if is_corr == (dom == "corrector"):
                traffic = k["dram_bytes_per_cell"] * cells
                tsrc = f"profiles/ncu_latest.json: {prof['report']}"
                ncu = {"fp64_pipe_pct": k.get("fp64_pipe_pct"), "issue_active_pct": k.get("issue_active_pct"),
                       "dram_throughput_pct": k.get("dram_throughput_pct"), "registers": k.get("registers"),
                       "warps_active_pct": k.get("warps_active_pct")}
    except Exception:
        pass
    b2k = sum(bytes_per_cell_update(ga, field))
    balg = 8 * (4 + ga + field) + 8 * (3 + ga)              # read U^n, z (+V, +n); write U^{n+1} (+V)
    r_fp = peak_gops * 1e9 / f_alg
    r_2k = min(hbm * 1e9 / b2k, r_fp)
    r_alg = min(hbm * 1e9 / balg, r_fp)
    hb = {"achieved": hbm_ach, "peak": hbm, "unit": "GB/s", "frac": frac_h, "peak_source": src}
    fb = {"achieved": fp_ach, "peak": peak_gops, "unit": "Gop/s (fp64 lane-ops)", "frac": frac_f,
          "ops_per_cell": ops_dom, "peak_note": f"148 SMs x 64 fp64 lanes x {peaks.get('sm_max_mhz', 1965.0):.0f} MHz"}
    b = hb if frac_h >= frac_f else fb
    return {"bound": "hbm" if frac_h >= frac_f else "alu", "achieved": b["achieved"], "peak": b["peak"],
            "unit": b["unit"], "frac": b["frac"], "traffic": traffic, "traffic_unit": "bytes/launch",
            "traffic_source": tsrc, "kernel": dom, "algorithmic_bytes": dom_bytes,
            "floors": {"hbm": hb, "fp64": fb}, "ncu": ncu,
            "step": {"R_2k": r_2k, "R_alg": r_alg, "B_2k": b2k, "B_alg": balg, "F_alg": f_alg,
                     "frac_R_2k": value / r_2k, "frac_R_alg": value / r_alg,
                     "R_2k_bound": "hbm" if hbm * 1e9 / b2k <= r_fp else "fp64",
                     "R_alg_bound": "hbm" if hbm * 1e9 / balg <= r_fp else "fp64"},
            "fp64_issue_ceiling": fp64_issue_ceiling(peak_gops)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--nx", type=int, default=None)
    ap.add_argument("--ny", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-crop", type=int, default=1024)
    ap.add_argument("--cpu-steps", type=int, default=12)
    ap.add_argument("--workload", default="swof", choices=("swof", "d8"))
    ap.add_argument("--shard-fused", action="store_true",
                    help="with --shard: fused exchange (kernels push boundary rows into the neighbours' "
                         "CUDA-IPC-mapped ghost rows) and in-stream NCCL barriers")
    ap.add_argument("--shard", action="store_true",
                    help="split the one grid into row strips over the ranks (strong scaling, NCCL halo exchange + "
                         "CFL all-reduce per step); the default for N > 1")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent full replicas (weak scaling) instead of the row-strip decomposition")
    ap.add_argument("--d8-dtype", default="f32", choices=("f32", "f64"))
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local = dist_env()
    from workloads import make
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if args.workload == "d8":
        return bench_d8(args, rank, world, local)
    if args.shard or args.shard_fused or (world > 1 and not args.replicas):
        return bench_shard(args, rank, world, local)

    import torch
    import torch.distributed as dist
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_1307_4839_b200 import Solver, params_from_config

    cfg = make(args.config, nx=args.nx, ny=args.ny)
    cells = cfg.nx * cfg.ny
    stream = torch.cuda.Stream()
    solver = Solver(params_from_config(cfg), cfg.z, cfg.fric_field, stream=stream)
    launches_per_step = solver.launches_per_step()
    v0 = cfg.vinf if cfg.ga is not None else None
    solver.set_state(cfg.h, cfg.hu, cfg.hv, v0, 0.0)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        return reduce_max(x, world, "cuda")

    # ---- device-resident throughput (value) ----
    solver.step(args.warmup)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0.record(stream)
        solver.step(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    value = aggregate_rate(world, cells, args.steps, ms)
    d = solver.diag()

    # ---- per-kernel device time (eager launches with events around each kernel) ----
    kp = min(args.steps, 20)
    ms_k = solver.step_profiled(kp)
    ms_pred, ms_corr = ms_k[0] / kp, ms_k[1] / kp

    # ---- end to end through the public API: pinned host state in, K steps, state out ----
    pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(cfg, k))).pin_memory() for k in ("h", "hu", "hv")}
    if cfg.ga is not None:
        pin["v"] = torch.from_numpy(np.ascontiguousarray(cfg.vinf)).pin_memory()
    outp = {k: torch.empty_like(v).pin_memory() for k, v in pin.items()}
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    solver.set_state(pin["h"], pin["hu"], pin["hv"], pin.get("v"), 0.0)
    solver.step(args.steps)
    solver.get_state(outp["h"], outp["hu"], outp["hv"], outp.get("v"))
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1))
    nfield = len(pin)
    io_bytes = nfield * cells * 8
    e2e = {"value": aggregate_rate(world, cells, args.steps, ms_e2e), "unit": UNIT,
           "h2d_bytes_per_step": io_bytes / args.steps, "d2h_bytes_per_step": io_bytes / args.steps,
           "ms_total": ms_e2e, "note": "set_state from pinned host + K steps + get_state to pinned host"}

    if rank != 0:
        solver.close()
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, src = load_peaks()
    ga, field = cfg.ga is not None, cfg.fric_field is not None
    bp, bc = bytes_per_cell_update(ga, field)
    dom = "corrector" if ms_corr >= ms_pred else "predictor"
    dom_ms = max(ms_corr, ms_pred)
    dom_bytes = (bc if dom == "corrector" else bp) * cells
    hbm_achieved = dom_bytes / (dom_ms / 1e3) / 1e9

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg4 recipe, SURVEY.md §8d)",
        "config": {"workload": args.config, "nx": cfg.nx, "ny": cfg.ny, "cells": cells,
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs (>=4.6 GB of fields) larger than L2; no flush"},
        "e2e": e2e,
        "gpu_launches": args.steps * launches_per_step,
        "kernels_ms": {"predictor": ms_pred, "corrector": ms_corr},
        "hbm": {"dominant_kernel": dom, "achieved_gbs": hbm_achieved, "peak_gbs": peaks["hbm_gbs"],
                "frac": hbm_achieved / peaks["hbm_gbs"], "bytes_per_cell_update": bp + bc, "peak_source": src},
        "clocks": clk.summary(),
        "diag": {"t": d["t"], "step": d["step"], "volume": d["volume"], "clamps": d["clamps"], "flags": d["flags"]},
    }

    fmax_mhz = peaks.get("sm_max_mhz", 1965.0)
    peak_gops = 148 * 64 * fmax_mhz * 1e6 / 1e9        # fp64 lane-ops/s: SMs x fp64 lanes x clock
    f_alg = None
    if not args.no_cpu_baseline:
        crop = min(args.cpu_crop, cfg.nx, cfg.ny)
        rate, cnt, secs, nst, host = cpu_sample(cfg, crop, args.cpu_steps)
        f_alg = f_alg_from_counters(cnt, cfg, nst, crop * crop)
        out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                               "sample": f"{crop}x{crop} centre crop of {args.config}, {nst} Heun steps, "
                                         f"walls, {secs:.1f} s single-threaded", **host}
    if f_alg is not None:
        out["roofline"] = roofline(peaks, src, peak_gops, f_alg, dom, dom_ms, dom_bytes, cells, value, ga, field)
    print(json.dumps(out), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()


def bench_shard(args, rank, world, local):
    """--shard: the workload's ONE grid cut into `world` row strips (the paper's MPI design,
    P:731-760), one per rank/GPU; per step two NCCL halo exchanges of 2 rows x 3 fields with each
    neighbour and one all-reduce(max) of the 2 CFL words.  Strong scaling: value = cells x steps / the
    slowest rank's time."""
    import torch
    import torch.distributed as dist
    from paper_1307_4839_b200.sharded import DistExchanger, IpcExchanger, ShardedSolver
    from workloads import make
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    cfg = make(args.config, nx=args.nx, ny=args.ny)
    cells = cfg.nx * cfg.ny
    stream = torch.cuda.Stream()
    if args.shard_fused:
        s = ShardedSolver(cfg, world, [rank], IpcExchanger(rank, world, in_stream=True), stream=stream, fused=True)
    else:
        s = ShardedSolver(cfg, world, [rank], DistExchanger(rank, world), stream=stream)
    s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
    s.step(args.warmup)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        s.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = reduce_max(e0.elapsed_time(e1), world, "cuda")
    # end to end: the host state in (every rank loads its strip), K steps, the state out
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
    s.step(args.steps)
    st = s.get_state()
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = reduce_max(e2.elapsed_time(e3), world, "cuda")
    s.close()
    if rank == 0:
        peaks, src = load_peaks()
        ga, field = cfg.ga is not None, cfg.fric_field is not None
        b2k = sum(bytes_per_cell_update(ga, field))
        ach = b2k * (cells / world) * args.steps / (ms / 1e3) / 1e9      # per rank (strip), whole step
        nfield = 3 + ga
        io = nfield * cells * 8
        out = {"metric": METRIC, "value": cells * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded cfg4 recipe, SURVEY.md §8d)",
               "config": {"workload": args.config, "nx": cfg.nx, "ny": cfg.ny, "cells": cells,
                          "parallelism": f"row strips x{world} (" + ("fused IPC halo push + NCCL barriers"
                                                                     if args.shard_fused else
                                                                     "NCCL halo exchange") + " + CFL all-reduce)",
                          "l2": "inputs larger than L2; no flush"},
               "gpu_launches": args.steps * (2 + (cfg.cfl_mode == "face")), "clocks": clk.summary(),
               "e2e": {"value": cells * args.steps / (ms_e2e / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": io / args.steps, "d2h_bytes_per_step": io / args.steps,
                       "note": "set_state of the host state into every strip + K steps + get_state"},
               "roofline": {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                            "frac": ach / peaks["hbm_gbs"], "traffic": None, "kernel": "whole step per strip",
                            "algorithmic_bytes_per_cell_update": b2k, "peak_source": src,
                            "note": "multi-GPU line: the step time includes the halo exchange; per-kernel "
                                    "fractions are on the N=1 line"},
               "t": st["t"], "step": st["step"]}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_d8(args, rank, world, local):
    """D8 flow direction on the paper's 14786 x 10086 DEM size, synthetic
    seeded raster (workloads/dem.py).  One "step" = one pass over the whole raster.  HBM-bound: the
    algorithmic bytes are one read of the raster and one code byte written per point."""
    import torch
    import torch.distributed as dist
    from paper_1307_4839_b200 import flow_direction
    from workloads.dem import DEM_SIZES, make_dem
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    nx, ny = DEM_SIZES["dem_large"]
    npts = nx * ny
    dtype = np.float32 if args.d8_dtype == "f32" else np.float64
    z = make_dem(nx, ny, dtype=dtype)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        zd = torch.from_numpy(z).cuda()
        out = torch.empty((ny, nx), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        flow_direction(zd, out, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()

    # device-resident: K passes, raster (>= 596 MB) larger than L2 -> no flush
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev[0].record(stream)
        for k in range(args.steps):
            flow_direction(zd, out, stream=stream)
            ev[k + 1].record(stream)
        torch.cuda.synchronize()
    barrier()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    ms = reduce_max(ev[0].elapsed_time(ev[-1]), world, "cuda")
    value = world * npts * args.steps / (ms / 1e3)
    # end to end: pinned host raster in, codes out, every step
    zp = torch.from_numpy(z).pin_memory()
    op = torch.empty((ny, nx), dtype=torch.uint8).pin_memory()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            zd.copy_(zp, non_blocking=True)
        flow_direction(zd, out, stream=stream)
        with torch.cuda.stream(stream):
            op.copy_(out, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = reduce_max(e0.elapsed_time(e1), world, "cuda")
    ok_codes = int(out.max().item()) <= 8
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks, src = load_peaks()
    bpp = z.itemsize + 1
    kern_ms = float(np.mean(per))
    ach = npts * bpp / (kern_ms / 1e3) / 1e9
    outj = {"metric": f"D8 flow-direction points/s ({args.d8_dtype} DEM, 1xB200)", "value": value, "unit": "points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak",
            # the paper's one D8 pass over a 14786 x 10086 DEM took 31 s with SkelGIS (101 s
            # with SkeTo) on unspecified CPU hardware: a comparison system on another
            # machine -- context only, not a baseline
            "vs_baseline": None,
            "context": {"paper_seconds_per_pass": 31.0, "system": "SkelGIS (SkeTo 101 s), unspecified CPU hardware",
                        "source": "BASELINE.md / PAPER.md:604-612", "ratio_to_paper_pass": value / (npts / 31.0)},
            "dtype": args.d8_dtype,
            "data": "synthetic (seeded sinusoid DEM, 1 cm quantised, no-data disc; workloads/dem.py)",
            "config": {"workload": "d8 dem_large", "nx": nx, "ny": ny, "points": npts,
                       "l2": f"raster {z.nbytes / 1e6:.0f} MB > L2; no flush"},
            "e2e": {"value": world * npts * args.steps / (ms_e2e / 1e3), "unit": "points/s",
                    "h2d_bytes_per_step": z.nbytes, "d2h_bytes_per_step": npts},
            "gpu_launches": args.steps,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": ach / peaks["hbm_gbs"], "traffic": None, "algorithmic_bytes_per_point": bpp,
                         "kernel": "d8_kernel", "peak_source": src},
            "clocks": clk.summary(), "codes_ok": ok_codes,
            "paper_context": "SkelGIS 31 s / SkeTo 101 s for this size on the paper's CPU cluster (P:604-612)"}
    if not args.no_cpu_baseline:
        import oracle
        t0 = time.perf_counter()
        ref = oracle.flow_direction(z)
        secs = time.perf_counter() - t0
        outj["cpu_baseline"] = {"value": npts / secs, "unit": "points/s", "cores": 1, "kind": "oracle",
                                "sample": f"the whole {nx}x{ny} raster, {secs:.1f} s single-threaded"}
        outj["parity_full_raster"] = bool(np.array_equal(ref, out.cpu().numpy()))
    print(json.dumps(outj), flush=True)
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, rank, world):
    """--impl reference: the oracle (plain single-threaded C), as it stands, on the host cores; each step
    is one Heun step on a bounded crop of the workload."""
    if rank != 0:
        return
    import oracle
    from workloads import make
    if args.workload == "d8":
        from workloads.dem import DEM_SIZES, make_dem
        nx, ny = DEM_SIZES["dem_large"]
        z = make_dem(nx, ny, dtype=np.float32 if args.d8_dtype == "f32" else np.float64)
        for _ in range(min(args.warmup, 1)):
            oracle.flow_direction(z)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.flow_direction(z)
        secs = time.perf_counter() - t0
        rate = nx * ny * args.steps / secs
        print(json.dumps({"metric": f"D8 flow-direction points/s ({args.d8_dtype} DEM, 1xB200)", "value": rate,
                          "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": secs * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": args.d8_dtype, "data": "synthetic",
                          "config": {"workload": "d8 dem_large", "nx": nx, "ny": ny}, "impl": "reference",
                          "cpu_baseline": {"value": rate, "unit": "points/s", "cores": 1, "kind": "oracle",
                                           "sample": f"the whole {nx}x{ny} raster per step"},
                          "e2e": {"value": rate, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                          "gpu_launches": 0}), flush=True)
        return
    cfg = make(args.config, nx=args.nx, ny=args.ny)
    crop = min(512, cfg.nx, cfg.ny)
    # warm-up then timed steps, each a single Heun step of the crop
    cpu_sample(cfg, crop, args.warmup)
    rate, cnt, secs, nst, host = cpu_sample(cfg, crop, args.steps)
    out = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": secs * 1e3 / max(nst, 1), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": args.config, "nx": cfg.nx, "ny": cfg.ny, "sample": f"{crop}x{crop} crop"},
           "impl": "reference",
           "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{crop}x{crop} centre crop of {args.config}, {nst} Heun steps", **host},
           "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
