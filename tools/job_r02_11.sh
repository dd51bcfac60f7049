# 4-GPU job: merged swaps (balanced partner order) correctness + A/B at 35 qubits
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "merged or four or trace" > gpurun_out/pytest_merged_n4.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -4 gpurun_out/pytest_merged_n4.log
if [ $rc -ne 0 ]; then exit 1; fi
run() { local label=$1; shift
  env "$@" timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 \
     bench.py --gpus 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload $WL > gpurun_out/n4_${label}.json 2> gpurun_out/n4_${label}.err
  echo "$label rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/n4_${label}.json').read().strip().splitlines()[-1]);print('$label', round(d['ms_per_step'],1), round(d.get('swap_ms_total') or 0,1), d.get('swap_exposed_frac'), d['config']['swaps'], d['config']['passes'])"
}
WL=qft:35 run qft35_merge1b QSV_MERGE_SWAPS=1
WL=random:35:20:2 run rnd35_merge1b QSV_MERGE_SWAPS=1
QSV_MERGE_SWAPS=1 timeout 600 python tools/trace_run.py random:30:20:2 4 gpurun_out/trace_rnd30_n4_merged.json 2>&1 | tail -1
QSV_MERGE_SWAPS=0 timeout 600 python tools/trace_run.py random:30:20:2 4 gpurun_out/trace_rnd30_n4_pairwise.json 2>&1 | tail -1
