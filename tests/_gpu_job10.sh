#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{
python - <<'PY'
import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg
c = pkg.Circuit.generate("uccsd:28:100000:3")
for cap in (512, 2048, 8192):
    t = time.time()
    e = pkg.Engine(c, pkg.PlanOptions(jit_max_kernels=cap))
    build = time.time() - t
    e.time(1, 0)
    ms = e.time(2, 0) / 2
    print("uccsd28 cap", cap, "passes", len(e.steps()), "jit", e.jit_info(), "build_s %.1f" % build, "ms/iter %.1f" % ms, flush=True)
    e.close()
PY
python tests/_prof_ab.py random:30:20:2 ""
QSV_TILE_NBUF=3 QSV_TILE_PD=1 python tests/_prof_ab.py random:30:20:2 ""
python tests/_prof_ab.py hea:30:5:4 ""
QSV_TILE_NBUF=3 QSV_TILE_PD=1 python tests/_prof_ab.py hea:30:5:4 ""
python tests/_prof_ab.py hea:33:5:4 ""
} 2>&1 | grep -v Warning | tee gpurun_out/ab6.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 700 gpurun_out/bench.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench N=2 rc=$?"; tail -c 500 gpurun_out/bench_n2.json
