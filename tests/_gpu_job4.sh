#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
python tests/_prof_ab.py random:30:20:2 relabel=0 relabel=2 relabel=2,min_low=6 relabel=2,min_low=7 relabel=0,min_low=6 relabel=0,min_low=7
QSV_PLAN_FIXED_L=1 python tests/_prof_ab.py random:30:20:2 relabel=0
python tests/_prof_ab.py hea:30:5:4 relabel=0 relabel=2 relabel=2,min_low=6
python tests/_prof_ab.py uccsd:26:30000:3 relabel=0 relabel=2 relabel=2,min_low=6
} 2>&1 | grep -v Warning | tee gpurun_out/ab.log
