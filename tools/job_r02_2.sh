cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "uccsd_full or uccsd28 or random30_full_size" --durations=10 > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_new.log
python tests/gpu_scripts/prof.py random:30:20:2 > gpurun_out/plain_h.log 2>&1; echo "prof rc=$?"; cat gpurun_out/plain_h.log
IDX=$(python - <<'PY'
import re
best = max(((float(m.group(2)), int(m.group(1))) for m in (re.match(r"(\d+) ([\d.]+) ms", l) for l in open("gpurun_out/plain_h.log")) if m))
print(best[1])
PY
)
echo "heaviest pass $IDX"
mkdir -p gpurun_out/jitsrc
QSV_JIT_DUMP=gpurun_out/jitsrc ncu --set full --import-source on --clock-control none -k regex:"qsv_jit|pass_kernel" -s $IDX -c 1 -o gpurun_out/r02_heavy python tests/gpu_scripts/prof.py random:30:20:2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
