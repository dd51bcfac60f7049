#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
for spec in random:30:20:2 qft:30 qaoa:30:2:1 hea:30:5:4 uccsd:24:20000:3; do
  python tests/_prof_ab.py $spec pass_budget=72.0 pass_budget=90.0 pass_budget=100.0 pass_budget=120.0
done
} 2>&1 | grep -v Warning | tee gpurun_out/ab4.log
