"""Per-source-line (outermost kernel-body line) ncu SASS instruction counts and stall samples of the stage kernels
(source line ranges of csrc/swof_kernels.cuh, via nvdisasm line info of the built library)."""
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
src = (ROOT / "paper_1307_4839_b200/csrc/swof_kernels.cuh").read_text().split("\n")
# phase markers: first source line containing the marker text starts the phase
markers = [("preamble", "const double t = st->t[par];"), ("P0 load", "// ---- P0:"), ("P1 xslopes", "// ---- P1:"),
           ("P2 xfaces", "// ---- P2:"), ("P3 xupdate", "// ---- P3:"), ("P4 yslopes", "// ---- P4:"),
           ("P5 yfaces", "// ---- P5:"), ("P6 cells", "// ---- P6:"), ("CFL reduce", "// warp-shuffle max on the u64")]
kstart = next(i for i, l in enumerate(src) if "__global__ void __launch_bounds__" in l) + 1
kend = next(i for i in range(kstart, len(src)) if src[i].startswith("}")) + 1
bounds = [(name, next(i for i in range(kstart, kend) if m in src[i - 1]) ) for name, m in markers]
def phase_of(line):
    if line is None or not (kstart <= line <= kend):
        return "helpers (inlined)"
    ph = "preamble"
    for name, b in bounds:
        if line >= b:
            ph = name
    return ph
# helpers called from phases are inlined: attribute by the innermost kernel-body line seen in the inline stack
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", str(ROOT / "paper_1307_4839_b200/libswof.so")], cwd=d, capture_output=True)
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
    if "## File" in l and "swof_kernels.cuh" in l:
        # inline info: '... line N inlined at "...", line M' -> keep the outermost kernel-body line
        nums = [int(x) for x in re.findall(r"line (\d+)", l)]
        body = [n for n in nums if kstart <= n <= kend]
        cur = body[-1] if body else (nums[0] if nums else None)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and func:
        lines[(func, int(m.group(1), 16))] = cur
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
kern = None
res = {}
for r in csv.reader(io.StringIO(sass)):
    if r and r[0] == "Kernel Name":
        kern = r[1]
        res[kern] = [collections.Counter(), collections.Counter()]
        base = None
        continue
    if r and r[0] == "Address":
        h = r
        continue
    if kern and len(r) > 5:
        a = int(r[0], 16)
        base = a if base is None else base
        fn = "_ZN4swof12stage_kernelILb%dEEEvNS_7KParamsENS_5KBufsEi" % (0 if "(bool)0" in kern else 1)
        ph = phase_of(lines.get((fn, a - base)))
        res[kern][0][ph] += int(r[h.index("# Samples")] or 0)
        res[kern][1][ph] += int(r[h.index("Instructions Executed")] or 0)
import json
for k, (smp, ins) in []:
    ts, ti = sum(smp.values()), sum(ins.values())
    print("==", k[:60])
    for ph in [b[0] for b in bounds] + ["helpers (inlined)"]:
        print(f"  {ph:18s} stall-samples {100 * smp[ph] / ts:5.1f}%   instructions {100 * ins[ph] / ti:5.1f}%")
# per-line
kern = None
per = {}
for r in csv.reader(io.StringIO(sass)):
    if r and r[0] == "Kernel Name":
        kern = r[1]; per[kern] = collections.defaultdict(lambda: [0, 0]); base = None; continue
    if r and r[0] == "Address":
        h = r; continue
    if kern and len(r) > 5:
        a = int(r[0], 16); base = a if base is None else base
        fn = "_ZN4swof12stage_kernelILb%dEEEvNS_7KParamsENS_5KBufsEi" % (0 if "(bool)0" in kern else 1)
        ln = lines.get((fn, a - base))
        per[kern][ln][0] += int(r[h.index("# Samples")] or 0)
        per[kern][ln][1] += int(r[h.index("Instructions Executed")] or 0)
for k, d in per.items():
    ts = sum(v[0] for v in d.values()); ti = sum(v[1] for v in d.values())
    print("==", k[:50])
    for ln, (s, i) in sorted(d.items(), key=lambda kv: -kv[1][1])[:40]:
        txt = src[ln - 1].strip()[:70] if ln else "?"
        print(f"  L{ln}: inst {100*i/ti:5.2f}% stall {100*s/ts:5.2f}%  {txt}")
