#!/bin/bash
# build + time kernel variants on the GPU box: bash tools/variants.sh "-DSWOF_MIN_BLOCKS=2" "-DSWOF_MIN_BLOCKS=3"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/variants.log
for v in "$@"; do
  python -m paper_1307_4839_b200.build --force $v > gpurun_out/build_var.log 2>&1 || { echo "$v build failed" >> gpurun_out/variants.log; continue; }
  regs=$(grep -E "registers|spill" gpurun_out/build_var.log | tr '\n' ' ' | cut -c1-400)
  out=$(timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1)
  echo "$v | $regs | $out" >> gpurun_out/variants.log
done
