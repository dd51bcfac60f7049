# 1-GPU job: pass budget / max_sweeps sweep with the round-2 kernels
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for spec in random:30:20:2 hea:30:5:4 qaoa:30:2:1 qft:30; do
  python tests/gpu_scripts/prof_ab.py $spec "pass_budget=100.0" "pass_budget=120.0" "pass_budget=140.0" "pass_budget=160.0" "pass_budget=200.0" "max_sweeps=6.0" "max_sweeps=10.0" 2>&1 | tee -a gpurun_out/budget_sweep_r02.log
done
python tests/gpu_scripts/prof_ab.py uccsd:24:20000:3 "pass_budget=100.0" "pass_budget=120.0" "pass_budget=160.0" 2>&1 | tee -a gpurun_out/budget_sweep_r02.log
