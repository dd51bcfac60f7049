#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
python3 - <<'PY' > /tmp/sb.py
src = open("tests/_swap_bench.py").read()
src = src.replace("for v in (l - 1, 10):", "for v in (l - 1,):").replace("for cl in (20, 22, 24, 26):", "for cl in (24, 26):").replace("for nbuf in (1, 2, 3):", "for nbuf in (2,):")
open("/tmp/sb.py", "w").write(src)
PY
cp /tmp/sb.py tests/_sb_tmp.py
for ENV in "X=1" "NCCL_P2P_NVL_CHUNKSIZE=4194304" "NCCL_MIN_NCHANNELS=32" "NCCL_NCHANNELS_PER_NET_PEER=32 NCCL_MIN_NCHANNELS=32" "NCCL_P2P_USE_CUDA_MEMCPY=1" "NCCL_P2P_LL_THRESHOLD=0 NCCL_MIN_NCHANNELS=16 NCCL_P2P_NVL_CHUNKSIZE=2097152"; do
  echo "== $ENV"
  env $ENV timeout 300 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tests/_sb_tmp.py 30 2>&1 | grep "GB/s"
done
