cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
N=$1
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_push_n$N.log 2>&1; echo "multi pytest rc=$?"; tail -3 gpurun_out/pytest_multi_push_n$N.log
big=$((33 + $(python -c "import math;print(int(math.log2($N)))")))
for wl in random:30:20:2 qft:$big random:$big:20:2; do
  for m in 0 2; do
    QSV_FUSE_SWAP=$m timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29525 \
      bench.py --gpus $N --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload $wl > gpurun_out/push_n${N}_${wl//:/_}_f$m.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/push_n${N}_${wl//:/_}_f$m.json').read().strip().splitlines()[-1]);print('$wl fuse=$m', round(d['ms_per_step'],1), round(d.get('swap_ms_total') or 0,1), d.get('swap_exposed_frac'), d['config']['swaps'], d.get('norm_error'))"
  done
done
