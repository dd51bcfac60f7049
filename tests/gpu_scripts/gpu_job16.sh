#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -3 gpurun_out/pytest_parity.log
{
for spec in qft:30 qaoa:30:2:1 random:30:20:2 qft:24; do
  python tests/gpu_scripts/prof_ab.py $spec ""
done
} 2>&1 | grep -v Warning | tee gpurun_out/ab12.log
