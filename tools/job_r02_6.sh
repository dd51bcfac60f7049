# 2-GPU job: full multi-GPU suite (trace, memory audit, shard files, cross-P, failure) + overlap traces
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_n2.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_multi_n2.log
for ov in 0 1; do
  QSV_OVERLAP=$ov timeout 600 python tools/trace_run.py qft:32 2 gpurun_out/trace_qft32_ov$ov.json 2>&1 | tail -2
  QSV_OVERLAP=$ov timeout 600 python tools/trace_run.py random:32:20:2 2 gpurun_out/trace_rnd32_ov$ov.json 2>&1 | tail -2
done
