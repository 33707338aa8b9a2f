"""Attribute ncu SASS stall samples (by reason) and executed instructions of the stage kernels to kernel
phases (source line ranges of csrc/swof_kernels.cuh, via nvdisasm line info of the built library).
Usage: python tools/ncu_phases.py <report.ncu-rep> [libswof.so] [swof_kernels.cuh]
(the library and source must be the ones the report was captured with)."""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rep = sys.argv[1]
so = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "paper_1307_4839_b200/libswof.so"
srcp = Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / "paper_1307_4839_b200/csrc/swof_kernels.cuh"
src = srcp.read_text().split("\n")
markers = [("preamble", "const double t = st->t[par];"), ("P0 load", "// ---- P0:"), ("P1 xslopes", "// ---- P1:"),
           ("P2 xfaces", "// ---- P2:"), ("P3 xupdate", "// ---- P3:"), ("P4 yslopes", "// ---- P4:"),
           ("P5 yfaces", "// ---- P5:"), ("P6 cells", "// ---- P6:"), ("CFL reduce", "// warp-shuffle max on the u64")]
kstart = next(i for i, l in enumerate(src) if "__global__ void __launch_bounds__" in l) + 1
kend = next(i for i in range(kstart, len(src)) if src[i].startswith("}")) + 1
bounds = [(name, next(i for i in range(kstart, kend) if m in src[i - 1])) for name, m in markers]


def phase_of(line):
    if line is None or not (kstart <= line <= kend):
        return "helpers (inlined)"
    ph = "preamble"
    for name, b in bounds:
        if line >= b:
            ph = name
    return ph


with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", str(so)], cwd=d, capture_output=True)
    cub = next(Path(d).glob("*.cubin"))
    dis = subprocess.run(["nvdisasm", "--print-line-info-inline", "-c", str(cub)], capture_output=True, text=True).stdout
lines = {}
func = None
cur = None
for l in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        func = m.group(1)
        continue
    if "## File" in l and srcp.name in l:
        nums = [int(x) for x in re.findall(r"line (\d+)", l)]
        body = [n for n in nums if kstart <= n <= kend]
        cur = body[-1] if body else (nums[0] if nums else None)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and func:
        lines[(func, int(m.group(1), 16))] = cur
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
REASONS = ["stall_wait", "stall_barrier", "stall_short_sb", "stall_long_sb", "stall_math", "stall_mio",
           "stall_branch_resolving", "stall_selected", "stall_not_selected", "stall_lg", "stall_dispatch"]
kern = None
res = {}
funcs = sorted({f for f, _ in lines})
for r in csv.reader(io.StringIO(sass)):
    if r and r[0] == "Kernel Name":
        kern = r[1]
        res[kern] = collections.defaultdict(collections.Counter)
        base = None
        continue
    if r and r[0] == "Address":
        h = r
        continue
    if kern and len(r) > 5:
        a = int(r[0], 16)
        base = a if base is None else base
        # the instance's mangled name from the template arguments in the demangled kernel name
        args = [int(x) for x in re.findall(r"\((?:bool|int)\)(\d+)", kern)]
        if len(args) == 5:
            fn = "_ZN4swof12stage_kernelILb%dENS_4PhysILi%dELb%dELb%dEEELb%dEEEvNS_7KParamsENS_5KBufsEi" % tuple(args)
        elif len(args) == 4:
            fn = "_ZN4swof12stage_kernelILb%dENS_4PhysILi%dELb%dELb%dEEEEEvNS_7KParamsENS_5KBufsEi" % tuple(args)
        else:
            fn = "_ZN4swof12stage_kernelILb%dEEEvNS_7KParamsENS_5KBufsEi" % args[0]
        ph = phase_of(lines.get((fn, a - base)))
        c = res[kern][ph]
        c["samples"] += int(r[h.index("# Samples")] or 0)
        c["inst"] += int(r[h.index("Instructions Executed")] or 0)
        for s in REASONS:
            c[s] += int(r[h.index(s)] or 0)
        for col, key in (("L1 Wavefronts Shared", "shwf"), ("L1 Wavefronts Shared Excessive", "shex")):
            try:
                c[key] += float(r[h.index(col)] or 0)
            except (ValueError, IndexError):
                pass
for k, phs in res.items():
    ts = sum(c["samples"] for c in phs.values())
    ti = sum(c["inst"] for c in phs.values())
    print("==", k[:70])
    tw = sum(c["shwf"] for c in phs.values()) or 1.0
    print(f"  {'phase':18s} {'inst%':>6s} {'smpl%':>6s} " + " ".join(f"{s[6:12]:>6s}" for s in REASONS) +
          "  shared-wavefronts% (excess%)")
    for ph in [b[0] for b in bounds] + ["helpers (inlined)"]:
        c = phs[ph]
        print(f"  {ph:18s} {100 * c['inst'] / ti:6.1f} {100 * c['samples'] / ts:6.1f} " +
              " ".join(f"{100 * c[s] / ts:6.1f}" for s in REASONS) +
              f"  {100 * c['shwf'] / tw:5.1f} ({100 * c['shex'] / tw:4.1f})")
