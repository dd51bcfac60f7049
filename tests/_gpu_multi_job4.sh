#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?" >> gpurun_out/pytest_multi.log
tail -3 gpurun_out/pytest_multi.log
run() {  # N tag env...
  N=$1; tag=$2; shift 2
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
    bench.py --gpus $N --steps 3 --warmup 3 --no-e2e > gpurun_out/bm_${tag}_n$N.json 2> gpurun_out/bm_${tag}_n$N.err
  python - "$N" "$tag" <<'PY'
import json, sys
N, tag = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/bm_{tag}_n{N}.json").read().strip().splitlines()[-1])
    print(tag, "N", N, "ms", round(d["ms_per_step"], 1), "swaps", d["config"]["swaps"], "swap_ms", round(d["swap_ms_total"], 1),
          "exposed", d.get("swap_exposed_frac"))
except Exception as e:
    print(tag, "N", N, "FAILED", e)
PY
}
for N in 2 4; do
  run $N ovl X=1
  run $N noovl QSV_OVERLAP=0
  run $N sms16 QSV_SWAP_SMS=16
  run $N sms32 QSV_SWAP_SMS=32
done
tail -5 gpurun_out/bm_ovl_n2.err
