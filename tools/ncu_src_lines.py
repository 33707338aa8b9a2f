"""Per-source-line ncu attribution of a kernel's SASS: instructions executed and stall samples by the
outermost line of the kernel body (the call site in KFILE) and by the innermost line (the helper).

    python tools/ncu_src_lines.py REPORT.ncu-rep LIB.so KFILE MANGLED_SUBSTR [NCU_KERNEL_REGEX [OPCODE_PREFIX]]

e.g. tools/ncu_src_lines.py gpurun_out/prof.ncu-rep paper_1307_4839_b200/libswof.so swof_march.cuh \
         march_kernelILb0ENS_4PhysILi1ELb1ELb0E 'march_kernel<\\(bool\\)0'
The library must be the one the report was captured with (SASS offsets are matched)."""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rep, lib, kfile, mangled = sys.argv[1:5]
kregex = sys.argv[5] if len(sys.argv) > 5 else None
opfilter = sys.argv[6] if len(sys.argv) > 6 else None      # count only SASS opcodes starting with this
srcs = {}


def src_line(f, n):
    if f not in srcs:
        p = next(ROOT.glob(f"**/csrc/{f}"), None)
        srcs[f] = p.read_text().split("\n") if p else []
    s = srcs[f]
    return s[n - 1].strip()[:80] if 0 < n <= len(s) else "?"


with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(lib).resolve())], cwd=d, capture_output=True)
    dis = ""
    for cub in Path(d).glob("*.cubin"):
        dis += subprocess.run(["nvdisasm", "--print-line-info-inline", "-c", str(cub)], capture_output=True,
                              text=True).stdout
info = {}
func = None
cur = (None, None)
for l in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        func = m.group(1) if mangled in m.group(1) else None
        continue
    if func is None:
        continue
    if "## File" in l:
        # '## File "a", line N [inlined at "b", line M ...]': innermost first
        pairs = re.findall(r'"([^"]+)", line (\d+)', l)
        pairs = [(Path(f).name, int(n)) for f, n in pairs]
        outer = [p for p in pairs if p[0] == kfile]
        cur = (outer[-1] if outer else None, pairs[0] if pairs else None, outer[0] if outer else None)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        info[int(m.group(1), 16)] = cur
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                      text=True).stdout
per_outer = collections.defaultdict(lambda: [0, 0])
per_inner = collections.defaultdict(lambda: [0, 0])
per_kin = collections.defaultdict(lambda: [0, 0])
kern, take, base = None, False, None
seen = set()
for r in csv.reader(io.StringIO(sass)):
    if r and r[0] == "Kernel Name":
        kern = r[1]
        # the page lists each kernel twice; count the first listing only
        take = (kregex is None or re.search(kregex, kern) is not None) and kern not in seen
        seen.add(kern)
        base = None
        continue
    if r and r[0] == "Address":
        h = r
        continue
    if take and len(r) > 5:
        a = int(r[0], 16)
        base = a if base is None else base
        o, i, k_in = info.get(a - base, (None, None, None))
        smp = int(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
        ins = int(r[h.index("Instructions Executed")] or 0)
        if opfilter:
            op = r[h.index("Source")].strip()
            op = op.split(None, 1)[1] if op.startswith("@") else op
            if not op.startswith(opfilter):
                continue
        per_outer[o][0] += smp
        per_outer[o][1] += ins
        per_inner[i][0] += smp
        per_inner[i][1] += ins
        per_kin[k_in][0] += smp
        per_kin[k_in][1] += ins
for title, d in (("call site (" + kfile + ")", per_outer), ("innermost line in " + kfile, per_kin),
                 ("innermost line", per_inner)):
    ts = sum(v[0] for v in d.values()) or 1
    ti = sum(v[1] for v in d.values()) or 1
    print(f"== by {title}: {ti} warp-instructions")
    for k, (s, i) in sorted(d.items(), key=lambda kv: -kv[1][1])[:32]:
        where = f"{k[0]}:{k[1]}" if k else "?"
        txt = src_line(*k) if k else ""
        print(f"  {where:24s} inst {100 * i / ti:5.2f}%  stall {100 * s / ts:5.2f}%  {txt}")
