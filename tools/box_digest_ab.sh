#!/bin/bash
# GPU box: the cfg4@100 and cfg3@500 full-size oracle digests side by side on the host cores (7 threads each)
# while the GPU runs an interleaved A/B of prebuilt libraries (arguments: the libraries, tools/ab_libs.sh)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/digest_on_box.sh cfg4@100 3300 7 > /dev/null 2>&1 &
bash tools/digest_on_box.sh cfg3@500 3300 7 > /dev/null 2>&1 &
ROUNDS=3 STEPS=60 bash tools/ab_libs.sh "$@"
tail -6 gpurun_out/ab_libs.log
wait
tail -3 gpurun_out/digest_cfg4@100.log gpurun_out/digest_cfg3@500.log
ls gpurun_out
