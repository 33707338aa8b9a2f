#!/bin/bash
# Interleaved A/B of prebuilt libraries (paths relative to the repo): ROUNDS=3 STEPS=60 bash tools/ab_libs.sh a.so b.so
# an entry lib.so@VAR=v,VAR2=w runs that library with those environment variables
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export SWOF_WORKLOAD_CACHE=/tmp/swof_wl_cache
: > gpurun_out/ab_libs.log
for r in $(seq 1 ${ROUNDS:-3}); do
  for lib in "$@"; do
    so=${lib%%@*}; envs=""; [ "$so" != "$lib" ] && envs=${lib#*@}
    v=$(env ${envs//,/ } SWOF_LIB=$PWD/$so timeout 600 python bench.py --steps ${STEPS:-60} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])" 2>/dev/null)
    echo "$lib $v" >> gpurun_out/ab_libs.log
  done
done
python - "$@" <<'PY'
import sys, statistics, collections
vals = collections.defaultdict(list)
for line in open("gpurun_out/ab_libs.log"):
    p = line.split()
    if len(p) == 2:
        try: vals[p[0]].append(float(p[1]))
        except ValueError: pass
with open("gpurun_out/ab_libs.log", "a") as f:
    for lib in sys.argv[1:]:
        v = vals.get(lib, [])
        f.write(f"lib {lib} median {statistics.median(v) if v else float('nan'):.4e} all {[f'{x:.4e}' for x in v]}\n")
PY
