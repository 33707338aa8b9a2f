#!/bin/bash
# GPU box: the >2^31-cell max-size case and cfg4@300, then one full-size oracle digest prefix (e.g. cfg3@2000)
# on all host cores but one, then that prefix's GPU full-size test against the digest just written.
#   bash tools/box_maxsize_digest_test.sh cfg3@2000 2900
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=tests/test_gpu_full_size.py::test_full_size_full_count
timeout 900 python -m pytest tests/test_gpu_max_size.py "$T[cfg4@300]" -m gpu -q -s \
  > gpurun_out/pytest_max.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_max.log
tail -4 gpurun_out/pytest_max.log
bash tools/digest_on_box.sh "$1" "${2:-2900}" $(( $(nproc) - 1 ))
if [ -f "gpurun_out/$1.npz" ]; then
  timeout 600 python -m pytest "$T[$1]" -m gpu -q -s > gpurun_out/pytest_$1.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_$1.log; tail -3 gpurun_out/pytest_$1.log
fi
