"""Summarise a gpurun_out/ profiling run into profiles/ (tracked).

Inputs (from tests/gpu_scripts/gpu_job.sh): gpurun_out/bench.json, bench_ref.json, launches.csv
(ncu --metrics gpu__time_duration.sum launch list of the bench command) and
prof_full.ncu-rep (ncu --set full of the heaviest pass).  Usage:
    python tests/gpu_scripts/mk_profiles.py r01 random:30:20:2
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
]


def launches(path):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    agg = {}
    for r in rd:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        if name.startswith("qsv_jit_"):
            name = "qsv_jit_* (NVRTC-specialised pass kernels)"
        ns = float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else (1e6 if r["Metric Unit"] == "ms" else 1))
        a = agg.setdefault(name, {"count": 0, "ms_total": 0.0})
        a["count"] += 1
        a["ms_total"] += ns / 1e6
    tot = sum(a["ms_total"] for a in agg.values())
    for a in agg.values():
        a["ms_total"] = round(a["ms_total"], 3)
        a["share"] = round(a["ms_total"] / tot, 4) if tot else 0.0
    return agg


def full_capture(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, u, v in zip(hdr, units, vals):
        if k in KEYS or k == "Kernel Name":
            d[k] = f"{v} {u}".strip()
    stalls = {}
    for k, v in zip(hdr, vals):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    d["stall_share_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:8]}
    return d


def gb(s):
    v, u = s.split()[:2] if len(s.split()) > 1 else (s, "byte")
    f = float(v)
    return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(u, 1)


def main():
    tag, workload = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    summ = {"workload": workload}
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        summ["launches"] = launches(os.path.join(OUT, "launches.csv"))
        shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches_{workload.replace(':', '_')}.csv"))
    if os.path.exists(os.path.join(OUT, "prof_full.ncu-rep")):
        fc = full_capture(os.path.join(OUT, "prof_full.ncu-rep"))
        summ["heaviest_pass_full_capture"] = fc
        rd, wr = gb(fc["dram__bytes_read.sum"]), gb(fc["dram__bytes_write.sum"])
        with open(os.path.join(PROF, "ncu_traffic.json"), "w") as f:
            json.dump({"workload": workload, "dram_bytes_per_launch": rd + wr,
                       "algorithmic_bytes_per_launch": 32 * (1 << int(workload.split(":")[1])),
                       "source": f"ncu --set full, heaviest pass of {workload} (profiles/{tag}_ncu_summary.json)"},
                      f, indent=1)
    with open(os.path.join(PROF, f"{tag}_ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    for src, dst in (("bench.json", f"{tag}_bench_{workload.replace(':', '_')}.json"),
                     ("bench_ref.json", f"{tag}_bench_reference.json")):
        p = os.path.join(OUT, src)
        if os.path.exists(p):
            shutil.copy(p, os.path.join(PROF, dst))
    print(json.dumps(summ, indent=1)[:3000])


if __name__ == "__main__":
    main()
