cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -k "fused" > gpurun_out/pytest_fused2.log 2>&1; rc=$?; echo "fused pytest rc=$rc"; tail -3 gpurun_out/pytest_fused2.log
[ $rc -ne 0 ] && exit 1
QSV_FUSE_SWAP=1 timeout 600 python tools/trace_run.py qft:32 2 gpurun_out/trace_qft32_fused2.json 2>&1 | tail -1
QSV_FUSE_SWAP=0 timeout 600 python tools/trace_run.py qft:32 2 gpurun_out/trace_qft32_plain2.json 2>&1 | tail -1
QSV_FUSE_SWAP=1 timeout 600 python tools/trace_run.py random:32:20:2 2 gpurun_out/trace_rnd32_fused2.json 2>&1 | tail -1
QSV_FUSE_SWAP=0 timeout 600 python tools/trace_run.py random:32:20:2 2 gpurun_out/trace_rnd32_plain2.json 2>&1 | tail -1
