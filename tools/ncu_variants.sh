#!/bin/bash
# ncu --set full of the stage kernels for several builds: bash tools/ncu_variants.sh ALT:v4 "-DX=1" ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xptxas -v -shared -Xcompiler -fPIC"
CMD="python bench.py --nx 4096 --ny 4096 --steps 4 --warmup 3 --no-cpu-baseline"
i=0
for v in "$@"; do
  i=$((i+1))
  if [[ $v == ALT:* ]]; then
    d=tools/alt/${v#ALT:}
    /usr/local/cuda/bin/nvcc $NVFLAGS -I $d -o paper_1307_4839_b200/libswof.so $d/swof.cu -lcudart > gpurun_out/build_nv$i.log 2>&1 || continue
  else
    python -m paper_1307_4839_b200.build --force $v > gpurun_out/build_nv$i.log 2>&1 || continue
  fi
  cp paper_1307_4839_b200/libswof.so gpurun_out/libswof_nv$i.so
  $CMD > gpurun_out/plain_nv$i.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"march_kernel" -s 6 -c 2 -o gpurun_out/prof_nv$i $CMD > gpurun_out/ncu_nv$i.log 2>&1
  echo "$i $v rc=$?" >> gpurun_out/ncu_variants.log
done
python -m paper_1307_4839_b200.build --force > /dev/null 2>&1
