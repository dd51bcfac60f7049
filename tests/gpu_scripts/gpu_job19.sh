#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -3 gpurun_out/pytest_parity.log
{
for spec in uccsd:26:30000:3 uccsd:24:20000:3; do
  python tests/gpu_scripts/prof_ab.py $spec ""
  QSV_JIT_FOLD_RELABEL=0 python tests/gpu_scripts/prof_ab.py $spec ""
done
python tests/gpu_scripts/prof_ab.py random:30:20:2 "" relabel=2
QSV_JIT_FOLD_RELABEL=0 python tests/gpu_scripts/prof_ab.py random:30:20:2 relabel=2
} 2>&1 | grep -v Warning | tee gpurun_out/ab15.log
