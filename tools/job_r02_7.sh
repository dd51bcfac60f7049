# 2-GPU job: fused-swap correctness first (bounded), then the multi suite, then 34-qubit A/B
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "fused" > gpurun_out/pytest_fused.log 2>&1; rc=$?; echo "fused pytest rc=$rc"; tail -5 gpurun_out/pytest_fused.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_n2.log 2>&1; echo "multi pytest rc=$?"; tail -4 gpurun_out/pytest_multi_n2.log
run() { local label=$1; shift
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
     bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload $WL > gpurun_out/bbop_${label}.json 2> gpurun_out/bbop_${label}.err
  echo "$label rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bbop_${label}.json').read().strip().splitlines()[-1]);print('$label', round(d['ms_per_step'],1), round(d.get('swap_ms_total'),1), d.get('swap_exposed_frac'), d['config']['swaps'], d['config']['passes'])"
}
WL=qft:34 run qft34_fuse0 QSV_FUSE_SWAP=0
WL=qft:34 run qft34_fuse1 QSV_FUSE_SWAP=1
WL=random:34:20:2 run rnd34_fuse0 QSV_FUSE_SWAP=0
WL=random:34:20:2 run rnd34_fuse1 QSV_FUSE_SWAP=1
QSV_FUSE_SWAP=1 timeout 600 python tools/trace_run.py qft:32 2 gpurun_out/trace_qft32_fused.json 2>&1 | tail -1
