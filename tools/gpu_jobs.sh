#!/usr/bin/env bash
# Reusable GPU jobs (run through gpurun; everything lands in gpurun_out/):
#   tools/gpu_jobs.sh suite            1 GPU: pytest -m gpu, smoke, bench + reference arm, ncu launch
#                                      list and a full capture of the heaviest pass (= tests/gpu_scripts/gpu_job.sh)
#   tools/gpu_jobs.sh multi N          N GPUs: the multi-GPU suite, then bench lines at N GPUs for
#                                      random-30 and (128 GiB per GPU) QFT-(32+log2 N) / random-(32+log2 N)
#   tools/gpu_jobs.sh ab "SPECS" "ENV1" "ENV2" ...   kernel-switch A/B (tools/env_ab.sh)
#   tools/gpu_jobs.sh fp64             measured DFMA / DMMA peaks (tools/fp64_peak.sh)
#   tools/gpu_jobs.sh trace SPEC N     PipelineTrace of one N-GPU run (tools/trace_run.py)
#   tools/gpu_jobs.sh dmmancu          ncu --set full of a pass with DMMA16 ops (QSV_DMMA_MIN_PIPE=32, random-28)
#   tools/gpu_jobs.sh fuseab N         N GPUs: the multi-GPU suite, then bench lines with separate
#                                      (QSV_FUSE_SWAP=0) and push-fused (=2) swaps, and traces of
#                                      QFT-32 / random-32 under 0, 1 (pull) and 2 (push) on 2 GPUs
#   tools/gpu_jobs.sh basisab N        N GPUs: the multi-GPU suite, then QFT bench lines with leading
#                                      swaps on the basis start moved (QSV_BASIS_SWAPS=0) or relabelled (=1)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
job=${1:-suite}; shift || true
case "$job" in
suite)
  bash tests/gpu_scripts/gpu_job.sh ;;
multi)
  N=${1:-2}
  timeout 2400 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_n$N.log 2>&1
  echo "multi pytest rc=$?"; tail -3 gpurun_out/pytest_multi_n$N.log
  big=$((32 + $(python -c "import math;print(int(math.log2($N)))")))
  for wl in random:30:20:2 qft:$big random:$big:20:2; do
    extra=""; [ "$wl" != "random:30:20:2" ] && extra="--no-e2e --no-cpu-baseline"
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29521 bench.py --gpus $N --steps 2 --warmup 3 $extra --workload $wl \
      > gpurun_out/n${N}_${wl//:/_}.json 2> gpurun_out/n${N}_${wl//:/_}.err
    echo "$wl rc=$?"; tail -c 400 gpurun_out/n${N}_${wl//:/_}.json
  done ;;
ab)
  ./tools/env_ab.sh "$@" 2>&1 | tee gpurun_out/ab.log ;;
fp64)
  ./tools/fp64_peak.sh ;;
trace)
  timeout 900 python tools/trace_run.py "$1" "${2:-2}" gpurun_out/trace.json ;;
dmmancu)
  QSV_DMMA_MIN_PIPE=32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:qsv_jit -c 1 \
    -o gpurun_out/dmma_pass python tests/gpu_scripts/prof.py random:28:20:2 > gpurun_out/dmmancu.log 2>&1
  echo "dmmancu rc=$?"; tail -3 gpurun_out/dmmancu.log ;;
fuseab)
  N=${1:-2}
  timeout 1800 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_n$N.log 2>&1
  echo "multi pytest rc=$?"; tail -3 gpurun_out/pytest_multi_n$N.log
  big=$((33 + $(python -c "import math;print(int(math.log2($N)))")))
  for wl in random:30:20:2 qft:$big random:$big:20:2; do
    for m in 0 2; do
      QSV_FUSE_SWAP=$m timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29525 bench.py --gpus $N --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload $wl \
        > gpurun_out/push_n${N}_${wl//:/_}_f$m.json 2>/dev/null
      python -c "import json;d=json.loads(open('gpurun_out/push_n${N}_${wl//:/_}_f$m.json').read().strip().splitlines()[-1]);print('$wl fuse=$m', round(d['ms_per_step'],1), d.get('swap_exposed_frac'), d['config']['swaps'], d.get('norm_error'))"
    done
  done
  if [ "$N" = 2 ]; then
    for spec in qft:32 random:32:20:2; do for m in 0 1 2; do
      QSV_FUSE_SWAP=$m timeout 600 python tools/trace_run.py $spec 2 gpurun_out/trace_${spec//:/_}_fuse$m.json 2>&1 | tail -1 | sed "s/^/[fuse=$m] /"
    done; done
  fi ;;
basisab)
  N=${1:-2}
  timeout 1800 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_multi_n$N.log 2>&1
  echo "multi pytest rc=$?"; tail -3 gpurun_out/pytest_multi_n$N.log
  big=$((33 + $(python -c "import math;print(int(math.log2($N)))")))
  for wl in qft:$big qft:30; do
    for b in 0 1; do
      QSV_BASIS_SWAPS=$b timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29527 bench.py --gpus $N --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-configs --workload $wl \
        > gpurun_out/basis_n${N}_${wl//:/_}_b$b.json 2>/dev/null
      python -c "import json;d=json.loads(open('gpurun_out/basis_n${N}_${wl//:/_}_b$b.json').read().strip().splitlines()[-1]);print('$wl basis_swaps=$b', round(d['ms_per_step'],1), d.get('swap_exposed_frac'), d['config']['swaps'], d.get('norm_error'))"
    done
  done ;;
*)
  echo "unknown job $job"; exit 2 ;;
esac
