#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
{
for spec in qft:30 qaoa:30:2:1 random:30:20:2 hea:30:5:4 uccsd:26:30000:3; do
  python tests/_prof_ab.py $spec relabel=1
  QSV_JIT_NO_EPI=1 python tests/_prof_ab.py $spec relabel=1
done
QSV_TILE_NBUF=3 QSV_TILE_PD=1 python tests/_prof_ab.py random:30:20:2 relabel=1
} 2>&1 | grep -v Warning | tee gpurun_out/ab2.log
