#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python tests/_prof_relabel.py random:30:20:2 > gpurun_out/prof_relabel.log 2>&1; echo "prof rc=$?"
grep total gpurun_out/prof_relabel.log
IDX=$(python - <<'PY'
rows=[l.split() for l in open("gpurun_out/prof_relabel.log") if l.startswith("2 ")]
# first relabel pass with one op
c=[int(r[1]) for r in rows if r[5]=="1" and r[4]=="1"]
print(c[0] if c else 0)
PY
)
echo "relabel pass $IDX"
cat > /tmp/one.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg
c = pkg.Circuit.generate("random:30:20:2")
e = pkg.Engine(c, pkg.PlanOptions(relabel=2)); e.set_basis(0); e.profile()
PY
ncu --set full --import-source on --clock-control none -k regex:"qsv_jit|pass_kernel" -s $IDX -c 1 -o gpurun_out/prof_relabel python /tmp/one.py > gpurun_out/ncu_relabel.log 2>&1; echo "ncu rc=$?"
