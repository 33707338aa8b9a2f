"""Static SASS opcode mix of one stage-kernel instance, grouped by kernel-body source line (nvdisasm
line info of the built library).  Usage: python tools/sass_static.py [mangled-name-substring] [line...]"""
import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
pat = sys.argv[1] if len(sys.argv) > 1 else "march_kernelILb0ENS_4PhysILi1ELb1ELb0E"
src = (ROOT / "paper_1307_4839_b200/csrc/swof_march.cuh").read_text().split("\n")
kstart = next(i for i, l in enumerate(src) if "__global__ void __launch_bounds__" in l) + 1
kend = next(i for i in range(kstart, len(src)) if src[i].startswith("}")) + 1
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", str(ROOT / "paper_1307_4839_b200/libswof.so")], cwd=d, capture_output=True)
    cub = next(Path(d).glob("*.cubin"))
    dis = subprocess.run(["nvdisasm", "--print-line-info-inline", "-c", str(cub)], capture_output=True, text=True).stdout
func = None
cur = None
by_line = collections.defaultdict(collections.Counter)
for l in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        func = m.group(1)
        continue
    if func is None or pat not in func:
        continue
    if "## File" in l and "swof_march.cuh" in l:
        nums = [int(x) for x in re.findall(r"line (\d+)", l)]
        body = [n for n in nums if kstart <= n <= kend]
        cur = body[-1] if body else (nums[0] if nums else None)
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", l)
    if m:
        by_line[cur][m.group(2)] += 1
tot = collections.Counter()
for c in by_line.values():
    tot.update(c)
print("total", sum(tot.values()), dict(tot.most_common(25)))
sel = [int(x) for x in sys.argv[2:]]
for ln, c in sorted(by_line.items(), key=lambda kv: -sum(kv[1].values()))[:25]:
    if sel and ln not in sel:
        continue
    txt = src[ln - 1].strip()[:60] if ln else "?"
    print(f"L{ln} n={sum(c.values())} {txt}\n    {dict(c.most_common(14))}")
