# 1-GPU job: race checks, CLI ablate/verify, default bench (with the other configs) and the reference arm
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_cli.py -q -m gpu -k "race_checks or cli" > gpurun_out/pytest_race_cli.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_race_cli.log
./paper_2509_04955_b200/lib/qsv verify > gpurun_out/qsv_verify.csv 2>&1; echo "verify rc=$?"; cat gpurun_out/qsv_verify.csv
./paper_2509_04955_b200/lib/qsv ablate --gen hea:28:5:4 --sizes 26,28 --repeat 2 --format csv > gpurun_out/qsv_ablate_hea.csv 2>&1; echo "ablate rc=$?"; cat gpurun_out/qsv_ablate_hea.csv | cut -c1-200
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 4000 gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.json
