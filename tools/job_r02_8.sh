# 1-GPU job: compute-sanitizer (racecheck, synccheck, memcheck) on every kernel flavour, then the full GPU suite
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export QSV_JIT_CACHE=/tmp/qsv_jit_san
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
QSV_DMMA_MIN_PIPE=1 timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize.py > gpurun_out/sanitizer_racecheck_dmma.log 2>&1; echo "racecheck dmma rc=$?"; tail -2 gpurun_out/sanitizer_racecheck_dmma.log
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu_full.log
