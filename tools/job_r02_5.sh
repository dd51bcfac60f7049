# 2-GPU job: multi-GPU parity suite, then BBOP region overlap A/B at 128 GiB per GPU
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_n2.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_multi_n2.log
run() { # $1 label, rest: env + args
  local label=$1; shift
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
     bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload $WL > gpurun_out/bbop_${label}.json 2> gpurun_out/bbop_${label}.err
  echo "$label rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bbop_${label}.json').read().strip().splitlines()[-1]);print('$label', d['ms_per_step'], d.get('swap_ms_total'), d.get('swap_exposed_frac'), d['config']['swaps'], d['config']['passes'])"
}
WL=qft:34 run qft34_off QSV_OVERLAP=0
WL=qft:34 run qft34_on QSV_OVERLAP=1
WL=random:34:20:2 run rnd34_off QSV_OVERLAP=0
WL=random:34:20:2 run rnd34_on QSV_OVERLAP=1
