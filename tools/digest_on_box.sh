#!/bin/bash
# Full-size oracle digest of one configuration on the GPU box's host cores, resumable across calls that land on
# the same box (the checkpoint lives in /tmp there): run from this container as
#   for i in 1 2 3; do gpurun --timeout 3600 -- bash tools/digest_on_box.sh cfg3 3200; [ -f gpurun_out/cfg3.npz ] && break; done
# (third argument: OpenMP threads, default nproc; two configurations side by side: 8 each on a 16-core host)
# then merge gpurun_out/digest_cfg3.json into tests/golden/full_size_digests.json (tools/merge_digest.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
name=$1; secs=${2:-3200}; threads=${3:-$(nproc)}
mkdir -p gpurun_out
ls -la /tmp/swof_ckpt 2>/dev/null >> gpurun_out/digest_${name}.log
OMP_NUM_THREADS=$threads python tools/oracle_digests.py $name --ckpt /tmp/swof_ckpt --max-seconds $secs >> gpurun_out/digest_${name}.log 2>&1
rc=$?
echo "rc=$rc" >> gpurun_out/digest_${name}.log
if [ $rc = 0 ]; then
  cp tests/golden/full_size/${name}.npz gpurun_out/${name}.npz
  python -c "import json,sys; d=json.load(open('tests/golden/full_size_digests.json')); json.dump({sys.argv[1]: d[sys.argv[1]]}, open('gpurun_out/digest_'+sys.argv[1]+'.json','w'), indent=1)" $name
fi
tail -3 gpurun_out/digest_${name}.log
