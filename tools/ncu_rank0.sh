#!/usr/bin/env bash
# torchrun --no-python tools/ncu_rank0.sh <bench args>: rank 0 runs bench.py under ncu (one
# capture of the first P2P swap kernel: NVLink and DRAM bytes), the other ranks plain.
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:p2p_swap -c 1 --csv --log-file "${NCU_LOG:-gpurun_out/ncu_swap.csv}" python bench.py "$@"
fi
exec python bench.py "$@"
