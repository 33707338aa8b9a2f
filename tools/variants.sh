#!/bin/bash
# build + time kernel variants on the GPU box:
#   bash tools/variants.sh "-DSWOF_MIN_BLOCKS=2" ...  (tools/ab.sh interleaves rounds: prefer it)
# "ALT:<name>" builds tools/alt/<name>/swof.cu (a frozen earlier kernel) instead of the tree's sources.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/variants.log
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xptxas -v -shared -Xcompiler -fPIC"
for v in "$@"; do
  if [[ $v == ALT:* ]]; then
    d=tools/alt/${v#ALT:}
    /usr/local/cuda/bin/nvcc $NVFLAGS -I $d -o paper_1307_4839_b200/libswof.so $d/swof.cu -lcudart > gpurun_out/build_var.log 2>&1 || { echo "$v build failed" >> gpurun_out/variants.log; continue; }
  else
    python -m paper_1307_4839_b200.build --force $v > gpurun_out/build_var.log 2>&1 || { echo "$v build failed" >> gpurun_out/variants.log; continue; }
  fi
  regs=$(grep -E "registers|spill" gpurun_out/build_var.log | tr '\n' ' ' | cut -c1-400)
  out=$(timeout 600 python bench.py --steps ${BENCH_STEPS:-30} --warmup 3 --no-cpu-baseline 2>&1 | tail -1)
  echo "$v | $regs | $out" >> gpurun_out/variants.log
done
python -m paper_1307_4839_b200.build --force > /dev/null 2>&1
