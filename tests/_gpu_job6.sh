#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
python tests/_prof_ab.py random:30:20:2 relabel=0 relabel=0,pass_budget=85.0 relabel=0,pass_budget=100.0 tile_k=12,relabel=0 tile_k=12,relabel=0,pass_budget=100.0 tile_k=12,relabel=0,pass_budget=130.0
QSV_TILE_NBUF=3 QSV_TILE_PD=1 python tests/_prof_ab.py random:30:20:2 relabel=0 relabel=0,pass_budget=100.0
python tests/_prof_ab.py qft:30 relabel=0 tile_k=12,relabel=0
python tests/_prof_ab.py qaoa:30:2:1 relabel=0 tile_k=12,relabel=0
python tests/_prof_ab.py hea:30:5:4 relabel=0 tile_k=12,relabel=0
python tests/_prof_ab.py uccsd:26:30000:3 relabel=1 tile_k=12,relabel=1 tile_k=12,relabel=0
python tests/_prof_ab.py hea:33:5:4 relabel=0
} 2>&1 | grep -v Warning | tee gpurun_out/ab3.log
