"""Summarise an ncu report: key metrics per kernel + SASS opcode mix (per cell)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else 4096 * 4096
json_out = sys.argv[3] if len(sys.argv) > 3 else None
summary = {"report": rep, "cells": cells, "kernels": {}}
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
for d in data:
    print("==", d[hdr.index("Kernel Name")][:60])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:66s} {d[i]:>18s} {units[i]}")
    name = d[hdr.index("Kernel Name")]
    def val(metric):
        return float(d[hdr.index(metric)].replace(",", "")) if metric in hdr and d[hdr.index(metric)] else None
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    def nbytes(metric):
        v = val(metric)
        return None if v is None else v * scale.get(units[hdr.index(metric)], 1.0)
    rb, wb = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    summary["kernels"][name] = {
        "duration_ms": val("gpu__time_duration.sum") * (1e-3 if units[hdr.index("gpu__time_duration.sum")] == "us" else 1.0),
        "dram_read_bytes": rb, "dram_write_bytes": wb, "dram_bytes_per_cell": (rb + wb) / cells,
        "fp64_pipe_pct": val("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": val("launch__registers_per_thread"),
        "dram_throughput_pct": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_clock_hz": val("sm__cycles_elapsed.avg.per_second") * 1e9 if units[hdr.index("sm__cycles_elapsed.avg.per_second")].lower().startswith("ghz") else val("sm__cycles_elapsed.avg.per_second"),
    }
    tot = sum(float(d[hdr.index(s)] or 0) for s in stalls)
    top = sorted(((float(d[hdr.index(s)] or 0), s) for s in stalls), reverse=True)[:8]
    print("  stalls:", ", ".join(f"{s.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for v, s in top))
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
kern = None
per = {}
for r in csv.reader(io.StringIO(sass)):
    if r and r[0] == "Kernel Name":
        kern = r[1]
        per[kern] = collections.Counter()
        continue
    if r and r[0] == "Address":
        h2 = r
        continue
    if kern and len(r) > 5:
        op = r[h2.index("Source")].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        per[kern][o.split(".")[0]] += int(r[h2.index("Instructions Executed")] or 0)
for k, c in per.items():
    tot = sum(c.values())
    print("==", k[:50], f"warp-inst/cell {tot / cells:.2f}")
    print("  " + ", ".join(f"{o} {n / cells:.2f}" for o, n in c.most_common(22)))
    for name in summary["kernels"]:
        corr = lambda n: re.search(r"_kernel<(\(bool\))?(1|true)\b", n) is not None
        if corr(name) == corr(k):
            summary["kernels"][name]["warp_inst_per_cell"] = tot / cells
            summary["kernels"][name]["opcode_mix_per_cell"] = {o: round(n / cells, 3) for o, n in c.most_common(30)}
if json_out:
    import json
    with open(json_out, "w") as f:
        json.dump(summary, f, indent=1)
