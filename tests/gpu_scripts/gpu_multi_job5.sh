#!/usr/bin/env bash
# Final multi-GPU numbers: random-30 strong scaling at N=2,4 (full bench line with e2e),
# then configs[4] shapes at the largest sizes a 4-GPU box holds (128 GiB per GPU).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) \
    bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  echo "bench N=$N rc=$?"; tail -c 400 gpurun_out/bench_n$N.json
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29610 + N)) \
    bench.py --gpus $N --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_n$N.json 2> gpurun_out/bench_ref_n$N.err
  echo "ref N=$N rc=$?"
done
for spec in qft:34 random:34:20:2; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29630 \
    bench.py --gpus 2 --steps 3 --warmup 3 --workload $spec --no-e2e --no-cpu-baseline > gpurun_out/bench_${spec//:/_}_n2.json 2> gpurun_out/bench_${spec//:/_}_n2.err
  echo "$spec N=2 rc=$?"; head -c 300 gpurun_out/bench_${spec//:/_}_n2.json; echo
done
for spec in qft:35 random:35:20:2; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 \
    bench.py --gpus 4 --steps 3 --warmup 3 --workload $spec --no-e2e --no-cpu-baseline > gpurun_out/bench_${spec//:/_}_n4.json 2> gpurun_out/bench_${spec//:/_}_n4.err
  echo "$spec N=4 rc=$?"; head -c 300 gpurun_out/bench_${spec//:/_}_n4.json; echo
done
