#!/usr/bin/env bash
# Measured FP64 peaks (DFMA, DMMA) with the SM clocks sampled during the run;
# writes profiles/fp64_peak.json (read by bench.py for the pass roofline).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
[ -x tools/fp64_peak ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/fp64_peak
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > gpurun_out/fp64_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak_raw.json
kill $SMI
python - <<'PY'
import json, statistics
d = json.load(open("gpurun_out/fp64_peak_raw.json"))
rows = [l.split(",") for l in open("gpurun_out/fp64_clocks.csv") if l.strip()]
sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
d["clocks"] = {"sm_mhz_median": statistics.median(sm) if sm else None,
               "sm_max_mhz": float(rows[0][1]) if rows else None,
               "power_w_max": max(float(r[2]) for r in rows) if rows else None,
               "samples": len(sm)}
json.dump(d, open("gpurun_out/fp64_peak.json", "w"))
print(json.dumps(d))
PY
