# 4-GPU job: merged-swap correctness, the multi-GPU suite, bench lines at 4 GPUs (random-30, QFT-35, random-35)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "merged or four" > gpurun_out/pytest_merged_n4.log 2>&1; rc=$?; echo "merged pytest rc=$rc"; tail -4 gpurun_out/pytest_merged_n4.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_n4.log 2>&1; echo "multi pytest rc=$?"; tail -4 gpurun_out/pytest_multi_n4.log
run() { local label=$1; shift
  env "$@" timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 \
     bench.py --gpus 4 --steps 2 --warmup 3 $EXTRA --workload $WL > gpurun_out/n4_${label}.json 2> gpurun_out/n4_${label}.err
  echo "$label rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/n4_${label}.json').read().strip().splitlines()[-1]);print('$label', round(d['ms_per_step'],1), round(d.get('swap_ms_total') or 0,1), d.get('swap_exposed_frac'), d['config']['swaps'], d['config']['passes'], d.get('e2e',{}) and d['e2e'].get('value'))"
}
EXTRA="" WL=random:30:20:2 run rnd30
EXTRA="--no-e2e --no-cpu-baseline" WL=qft:35 run qft35_merge1 QSV_MERGE_SWAPS=1
EXTRA="--no-e2e --no-cpu-baseline" WL=qft:35 run qft35_merge0 QSV_MERGE_SWAPS=0
EXTRA="--no-e2e --no-cpu-baseline" WL=random:35:20:2 run rnd35_merge1 QSV_MERGE_SWAPS=1
EXTRA="--no-e2e --no-cpu-baseline" WL=random:35:20:2 run rnd35_merge0 QSV_MERGE_SWAPS=0
