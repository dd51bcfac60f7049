#!/usr/bin/env bash
# Parity + bench after a planner/kernel change (one GPU).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json | head -c 600; echo
for spec in uccsd:28:100000:3 hea:30:5:4 qft:30 qaoa:30:2:1; do
  python bench.py --no-cpu-baseline --no-e2e --workload $spec --steps 3 --warmup 3 > gpurun_out/bench_${spec//:/_}.json 2>>gpurun_out/bench.err; echo "$spec rc=$?"
done
