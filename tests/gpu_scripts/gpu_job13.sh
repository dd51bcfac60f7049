#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
{
for spec in random:30:20:2 hea:30:5:4 qaoa:30:2:1 qft:30 uccsd:24:20000:3; do
  python tests/gpu_scripts/prof_ab.py $spec ""
  QSV_TMA_SPREAD=0 python tests/gpu_scripts/prof_ab.py $spec ""
done
} 2>&1 | grep -v Warning | tee gpurun_out/ab9.log
