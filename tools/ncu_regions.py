"""Per-region attribution of a marching-kernel capture, from the SASS in the ncu report itself (no library
needed): the steady-state row loop (the largest backward branch) is cut at its warp votes (VOTE.ANY: the
slow-path votes that close the scheduling regions), and the instructions executed and stall
samples are summed per region; the code outside the loop is one more line.

    python tools/ncu_regions.py REPORT.ncu-rep KERNEL_REGEX
e.g. python tools/ncu_regions.py gpurun_out/prof8k.ncu-rep 'march_kernel<1'
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kregex = sys.argv[1], sys.argv[2]
page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows, take, seen, hdr = [], False, set(), None
for r in csv.reader(io.StringIO(page)):
    if r and r[0] == "Kernel Name":
        take = re.search(kregex, r[1]) is not None and r[1] not in seen and not rows
        seen.add(r[1])
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if take and hdr and len(r) > 5:
        rows.append((int(r[0], 16), r[hdr.index("Source")].strip(),
                     int(r[hdr.index("Instructions Executed")] or 0),
                     int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
if not rows:
    sys.exit("kernel not found")
addr = {a: k for k, (a, *_rest) in enumerate(rows)}
best = None
for k, (a, src, _, _) in enumerate(rows):
    m = re.search(r"\bBRA\b[^0-9a-fx]*(0x[0-9a-f]+)", src)
    if m:
        t = int(m.group(1), 16)
        if t < a and t in addr and (best is None or k - addr[t] > best[1] - best[0]):
            best = (addr[t], k)
tot_i = sum(r[2] for r in rows) or 1
tot_s = sum(r[3] for r in rows) or 1
lo, hi = best
cuts = [k for k in range(lo, hi + 1) if "VOTE.ANY" in rows[k][1]]
bounds = [lo] + [c + 1 for c in cuts] + [hi + 1]
names = ["fetch + primitives + y stencil + y face", "x stencil + x face", "update + sources"]
names += (["Heun + CFL speeds", "after the last vote (stores, loop control, what ptxas placed there)"] if len(cuts) >= 4 else ["after the last vote (stores, loop control, what ptxas placed there)"])
names += [f"region {i}" for i in range(len(names), 20)]
print(f"== {kregex}: loop {hex(rows[lo][0])}-{hex(rows[hi][0])}, {len(cuts)} votes")
for i in range(len(bounds) - 1):
    seg = rows[bounds[i]:bounds[i + 1]]
    ni = sum(r[2] for r in seg)
    ns = sum(r[3] for r in seg)
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", r[1]).split()[0].split(".")[0] for r in seg if r[2])
    fp = sum(r[2] for r in seg if re.sub(r"^@!?U?P\w+\s+", "", r[1]).split()[0].split(".")[0]
             in ("DADD", "DMUL", "DFMA", "DSETP"))
    print(f"  {names[i]:42s} inst {100 * ni / tot_i:5.1f}%  stall {100 * ns / tot_s:5.1f}%  fp64 share of its "
          f"instructions {100 * fp / max(ni, 1):4.1f}%")
outside = [r for k, r in enumerate(rows) if k < lo or k > hi]
print(f"  {'outside the row loop':42s} inst {100 * sum(r[2] for r in outside) / tot_i:5.1f}%  "
      f"stall {100 * sum(r[3] for r in outside) / tot_s:5.1f}%")
