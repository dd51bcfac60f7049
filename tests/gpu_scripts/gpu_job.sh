#!/usr/bin/env bash
# One gpurun job: GPU tests, bench, ncu launch list + one full capture of the heaviest pass.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra-configs"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tests/gpu_scripts/prof.py random:30:20:2 > gpurun_out/plain_h.log 2>&1 && \
IDX=$(python - <<'PY'
import re
best = max(((float(m.group(2)), int(m.group(1))) for m in (re.match(r"(\d+) ([\d.]+) ms", l) for l in open("gpurun_out/plain_h.log")) if m))
print(best[1])
PY
) && echo "heaviest pass $IDX" && \
ncu --set full --import-source on --clock-control none -k regex:"qsv_jit|pass_kernel" -s $IDX -c 1 -o gpurun_out/prof_full python tests/gpu_scripts/prof.py random:30:20:2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tests/gpu_scripts/prof.py hea:33:5:4 > gpurun_out/prof_hea33.log 2>&1; echo "prof hea33 rc=$?"; tail -2 gpurun_out/prof_hea33.log
tail -2 gpurun_out/plain_h.log
