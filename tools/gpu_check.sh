#!/bin/bash
# GPU pass: [tests] [bench] [ncu]   e.g. bash tools/gpu_check.sh tests bench ncu
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for what in "$@"; do
case $what in
tests) timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log ;;
quick) timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -x -k "one_step or predictor or 3x3" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log ;;
bench) timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log ;;
ncu)
CMD="python bench.py --nx 4096 --ny 4096 --steps 4 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"march_kernel" -s 6 -c 2 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log ;;
launches)
CMD="python bench.py --nx 4096 --ny 4096 --steps 4 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_list.log ;;
esac
done
# full-size variants (the bench's own launch configuration)
for what in "$@"; do
case $what in
ncu8k)
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain8k.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches8k.csv $CMD > gpurun_out/ncu_list8k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"march_kernel" -s 6 -c 2 -o gpurun_out/prof8k $CMD > gpurun_out/ncu_full8k.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full8k.log ;;
esac
done
