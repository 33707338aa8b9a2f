"""Static SASS of the steady-state row loop of one stage-kernel instance: the largest backward branch's body,
its instruction count and opcode mix (what one marching row costs per lane), plus registers and spills.
Usage: python tools/sass_loop.py lib.so [mangled-name-substring] [--dump]"""
import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

so = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "march_kernelILb1ENS_4PhysILi1ELb1ELb0EEELb0ELb0E"
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(so).resolve())], cwd=d, capture_output=True)
    cub = next(Path(d).glob("*.cubin"))
    dis = subprocess.run(["nvdisasm", "-c", str(cub)], capture_output=True, text=True).stdout
func, ins, labels, pending = None, [], {}, []
for l in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        func = m.group(1)
        continue
    if func is None or pat not in func:
        continue
    m = re.match(r"\s*(\.L_x_\d+):", l)
    if m:
        pending.append(m.group(1))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        a = int(m.group(1), 16)
        for lb in pending:
            labels[lb] = a
        pending = []
        ins.append((a, m.group(2).strip()))
if not ins:
    sys.exit(f"no function matching {pat}")
addr = {a: k for k, (a, _) in enumerate(ins)}
best = None
for k, (a, txt) in enumerate(ins):
    m = re.search(r"\bBRA\b.*?\((\.L_x_\d+)\)", txt)
    if m and m.group(1) in labels:
        tgt = labels[m.group(1)]
        if tgt < a and tgt in addr and (best is None or k - addr[tgt] > best[1] - best[0]):
            best = (addr[tgt], k)
lo, hi = best
body = ins[lo:hi + 1]
mix = collections.Counter()
for _, txt in body:
    op = re.sub(r"^@!?U?P\w+\s+", "", txt).split()[0].split(".")[0]
    mix[op] += 1
fp64 = sum(v for k, v in mix.items() if k in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"))
print(f"{pat}: whole function {len(ins)} instructions; loop body {len(body)} instructions, fp64 {fp64}, "
      f"branches {mix['BRA']}")
print("  " + ", ".join(f"{k} {v}" for k, v in mix.most_common(24)))
if "--dump" in sys.argv:
    for a, t in body:
        print(f"{a:06x} {t}")
