#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
python tests/gpu_scripts/prof_ab.py hea:33:5:4 ""
python tests/gpu_scripts/prof_ab.py uccsd:28:100000:3 ""
python tests/gpu_scripts/prof_ab.py qft:24 ""
python tests/gpu_scripts/prof_ab.py random:30:20:2 fusion=0,multi_op_passes=0
} 2>&1 | grep -v Warning | tee gpurun_out/ab13.log
