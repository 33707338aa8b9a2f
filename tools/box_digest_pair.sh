cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nproc > gpurun_out/box_host.txt; free -g >> gpurun_out/box_host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core" >> gpurun_out/box_host.txt
bash tools/gpu_check.sh tests bench
tail -2 gpurun_out/pytest_gpu.log; tail -c 300 gpurun_out/bench.log
bash tools/digest_on_box.sh cfg4 11000 8 > /dev/null 2>&1 &
bash tools/digest_on_box.sh cfg3 11000 8 > /dev/null 2>&1 &
wait
tail -3 gpurun_out/digest_cfg4.log gpurun_out/digest_cfg3.log
ls -la gpurun_out
