#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
python tests/gpu_scripts/prof_ab.py uccsd:26:30000:3 "" relabel=0 relabel=2
python tests/gpu_scripts/prof_ab.py uccsd:24:20000:3 "" relabel=0 relabel=2
} 2>&1 | grep -v Warning | tee gpurun_out/ab14.log
