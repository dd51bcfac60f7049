#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
for spec in random:30:20:2 hea:30:5:4 qaoa:30:2:1 qft:30; do
  python tests/gpu_scripts/prof_ab.py $spec pass_budget=100.0 pass_budget=120.0 pass_budget=140.0 pass_budget=170.0 max_sweeps=10.0 pass_budget=140.0,max_sweeps=10.0
done
} 2>&1 | grep -v Warning | tee gpurun_out/ab11.log
