#!/bin/bash
# GPU box: the GPU suite + bench, then one full-size oracle digest prefix (e.g. cfg4@300) on all host cores
# but one, within one call's hour: bash tools/box_suite_digest.sh cfg4@300 2700
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nproc > gpurun_out/box_host.txt
bash tools/gpu_check.sh tests bench
tail -2 gpurun_out/pytest_gpu.log; tail -c 400 gpurun_out/bench.log
bash tools/digest_on_box.sh "$1" "${2:-2700}" $(( $(nproc) - 1 ))
ls gpurun_out
