#!/bin/bash
# GPU box: one full-size oracle digest on all host cores but one (e.g. cfg3@2000), within one call's hour
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/digest_on_box.sh "$1" "${2:-3300}" $(( $(nproc) - 1 ))
ls gpurun_out
