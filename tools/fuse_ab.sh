#!/usr/bin/env bash
# 2-GPU fused-swap check and A/B: pull (QSV_FUSE_SWAP=1), push (=2) against plain swaps (=0)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "fused" > gpurun_out/pytest_fused.log 2>&1; rc=$?; echo "fused pytest rc=$rc"; tail -3 gpurun_out/pytest_fused.log
[ $rc -ne 0 ] && exit 1
for spec in qft:32 random:32:20:2; do
  for m in 0 1 2; do
    QSV_FUSE_SWAP=$m timeout 600 python tools/trace_run.py $spec 2 gpurun_out/trace_${spec//:/_}_fuse$m.json 2>&1 | tail -1 | sed "s/^/[fuse=$m] /"
  done
done
