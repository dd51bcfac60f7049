#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
for spec in random:30:20:2 qaoa:30:2:1; do
  python tests/gpu_scripts/prof_ab.py $spec ""
  QSV_TILE_NBUF=3 QSV_TILE_PD=1 python tests/gpu_scripts/prof_ab.py $spec ""
  QSV_JIT_SPLIT=1 python tests/gpu_scripts/prof_ab.py $spec ""
done
} 2>&1 | grep -v Warning | tee gpurun_out/ab10.log
