#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?" >> gpurun_out/pytest_multi.log
tail -3 gpurun_out/pytest_multi.log
for N in 2 4; do
  for MODE in p2p nccl; do
    QSV_SWAP_MODE=$MODE timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tests/_swap_bench3.py $((30 - N / 2)) 2>&1 | grep "mode="
  done
done
run() {  # N tag env...
  N=$1; tag=$2; shift 2
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
    bench.py --gpus $N --steps 3 --warmup 3 --no-e2e > gpurun_out/bm_${tag}_n$N.json 2> gpurun_out/bm_${tag}_n$N.err
  python - "$N" "$tag" <<'PY'
import json, sys
N, tag = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/bm_{tag}_n{N}.json").read().strip().splitlines()[-1])
print(tag, "N", N, "ms", round(d["ms_per_step"], 1), "swaps", d["config"]["swaps"], "swap_ms", round(d["swap_ms_total"], 1),
      "exposed", d.get("swap_exposed_frac"))
PY
}
for N in 2 4; do
  run $N p2p X=1
  run $N nccl QSV_SWAP_MODE=nccl
done
