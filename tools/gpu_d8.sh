#!/bin/bash
# GPU pass for the D8 flow direction: tests, bench line, ncu launch list + full capture of d8_kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_d8.py -m gpu -q > gpurun_out/pytest_d8.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d8.log
timeout 600 python bench.py --workload d8 --steps 20 --warmup 5 > gpurun_out/bench_d8.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_d8.log
timeout 600 python bench.py --workload d8 --d8-dtype f64 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_d8_f64.log 2>&1
CMD="python bench.py --workload d8 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_d8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"d8_kernel|d8_march_kernel" -s 3 -c 1 -o gpurun_out/prof_d8 $CMD > gpurun_out/ncu_d8.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_d8.log
