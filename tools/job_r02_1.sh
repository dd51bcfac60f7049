cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
./tools/fp64_peak.sh > gpurun_out/fp64.log 2>&1; echo "fp64 rc=$?"; tail -1 gpurun_out/fp64.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "uccsd_full or uccsd28 or random30_full_size" --durations=10 > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_new.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_ref.json
