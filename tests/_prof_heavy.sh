#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
python tests/_prof.py random:30:20:2 > gpurun_out/plain_h.log 2>&1 || exit 1
python - <<'PY' > gpurun_out/heavy_idx.txt
import re
best = max(((float(m.group(2)), int(m.group(1))) for m in (re.match(r"(\d+) ([\d.]+) ms", l) for l in open("gpurun_out/plain_h.log")) if m))
print(best[1])
PY
IDX=$(cat gpurun_out/heavy_idx.txt)
echo "heaviest pass index $IDX"
ncu --set full --import-source on --clock-control none -k regex:pass_kernel -s $IDX -c 1 -o gpurun_out/prof_heavy python tests/_prof.py random:30:20:2 > gpurun_out/ncu_h.log 2>&1; echo "ncu rc=$?"
