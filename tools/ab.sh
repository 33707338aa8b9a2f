#!/bin/bash
# Interleaved A/B timing of kernel builds on the GPU box (reduces box/clock drift):
#   ROUNDS=3 STEPS=60 bash tools/ab.sh "" "-DFOO=1" ...
# every variant is built once into gpurun_out/ab_<i>.so, then the rounds run the variants in turn;
# prints each variant's values and median (cell-updates/s).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/ab.log
export SWOF_WORKLOAD_CACHE=/tmp/swof_wl_cache
i=0
for v in "$@"; do
  # a variant is "-DNAME=V ..." defines, optionally with nvcc flags after "::" ("-DX=1 :: -Xptxas -dlcm=cg")
  defs="${v%%::*}"; extra=""; [[ "$v" == *::* ]] && extra="${v#*::}"
  SWOF_NVCC_EXTRA="$extra" python -m paper_1307_4839_b200.build --force $defs > gpurun_out/ab_build_$i.log 2>&1 || echo "variant $i build failed" >> gpurun_out/ab.log
  cp paper_1307_4839_b200/libswof.so gpurun_out/ab_$i.so
  i=$((i+1))
done
n=$i
for r in $(seq 1 ${ROUNDS:-3}); do
  for i in $(seq 0 $((n-1))); do
    cp gpurun_out/ab_$i.so paper_1307_4839_b200/libswof.so
    val=$(timeout 600 python bench.py --steps ${STEPS:-60} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])" 2>/dev/null)
    echo "$i $val" >> gpurun_out/ab.log
  done
done
python - "$@" <<'PY'
import sys, statistics, collections
vals = collections.defaultdict(list)
for line in open("gpurun_out/ab.log"):
    p = line.split()
    if len(p) == 2 and p[0].isdigit():
        try: vals[int(p[0])].append(float(p[1]))
        except ValueError: pass
with open("gpurun_out/ab.log", "a") as f:
    for i, name in enumerate(sys.argv[1:]):
        v = vals.get(i, [])
        f.write(f"variant {i} [{name}] median {statistics.median(v) if v else float('nan'):.4e} all {[f'{x:.4e}' for x in v]}\n")
PY
rm -f gpurun_out/ab_*.so
python -m paper_1307_4839_b200.build --force > /dev/null 2>&1
