#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?" >> gpurun_out/pytest_multi.log
tail -3 gpurun_out/pytest_multi.log
for spec in qft:34; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29630 \
    bench.py --gpus 2 --steps 3 --warmup 3 --workload $spec --no-e2e --no-cpu-baseline > gpurun_out/bench_${spec//:/_}_n2.json 2> gpurun_out/bench_${spec//:/_}_n2.err
  echo "$spec N=2 rc=$?"; head -c 300 gpurun_out/bench_${spec//:/_}_n2.json; echo
done
for spec in qft:35; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 \
    bench.py --gpus 4 --steps 3 --warmup 3 --workload $spec --no-e2e --no-cpu-baseline > gpurun_out/bench_${spec//:/_}_n4.json 2> gpurun_out/bench_${spec//:/_}_n4.err
  echo "$spec N=4 rc=$?"; head -c 300 gpurun_out/bench_${spec//:/_}_n4.json; echo
done
