#!/usr/bin/env bash
# Multi-GPU job (gpurun --gpus 4): NCCL parity tests, then the torchrun bench at N=2 and N=4.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?" >> gpurun_out/pytest_multi.log
tail -3 gpurun_out/pytest_multi.log
for N in 2 4; do
  [ "$N" -le "$NG" ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N \
    bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
  echo "bench N=$N rc=$?"; head -c 400 gpurun_out/bench_n$N.json; echo
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_n$N.json 2> gpurun_out/bench_ref_n$N.err
  echo "ref N=$N rc=$?"
done
