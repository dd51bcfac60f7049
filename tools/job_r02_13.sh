# 1-GPU job: tensor-map tile copies: parity subset + race checks + A/B
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "generated_circuits or config_shapes or random_mnemonic or single_gate or qft24 or mirror_full or dense_unitaries or race" > gpurun_out/pytest_tma.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -3 gpurun_out/pytest_tma.log
./tools/env_ab.sh "random:30:20:2 hea:30:5:4 qft:30 uccsd:24:20000:3 qaoa:30:2:1 hea:33:5:4" "QSV_TMA_TENSOR=0" "QSV_TMA_TENSOR=1" 2>&1 | tee gpurun_out/ab_tma.log
python tests/gpu_scripts/prof.py random:30:20:2 > gpurun_out/prof_tma.log 2>&1; tail -37 gpurun_out/prof_tma.log
