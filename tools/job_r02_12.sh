# 1-GPU job: literal-matrix kernels: parity subset + A/B
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "generated_circuits or config_shapes or random_mnemonic or single_gate or qft24 or mirror_full" > gpurun_out/pytest_lit.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_lit.log
./tools/env_ab.sh "random:30:20:2 hea:30:5:4 qft:30 uccsd:24:20000:3 qaoa:30:2:1" "QSV_JIT_LITERALS=0" "QSV_JIT_LITERALS=1" 2>&1 | tee gpurun_out/ab_lit.log
python tests/gpu_scripts/prof.py random:30:20:2 > gpurun_out/prof_lit.log 2>&1; tail -38 gpurun_out/prof_lit.log
