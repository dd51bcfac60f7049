#!/usr/bin/env python3
"""Benchmark of the B200 state-vector hot path (arXiv 2509.04955 north star).

One step = one full simulation of the workload circuit from |0...0> (state
initialisation + every fused pass / swap of the planned program) on an
HBM-resident state.  Default workload: BASELINE.json configs[1], the random
30-qubit depth-20 H/RX/RZ/CNOT circuit with gate contraction (DAGC) on.

Metric (BASELINE.json): circuit time, gates/s and HBM GB/s; `value` = gates/s
(gates after QASM lowering, before fusion) of the whole job, device-timed with
CUDA events on the engine stream, max over ranks.

  python bench.py                          # N=1, default K/W
  torchrun --nproc-per-node N bench.py --gpus N   # N ranks, strong scaling
  python bench.py --impl reference         # reference CPU path on host cores

Everything measured here runs through libqsv.so / libqsim.so; the CPU legs
(`cpu_baseline`, `--impl reference`) run the oracle restatement (oracle/).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

HBM_FALLBACK_GBS = 6650.0
F64_NOMINAL_TFLOPS = 37.0  # B200 FP64 datasheet figure; used only when the measured file is absent


def load_f64_peak() -> tuple[float, str]:
    """The FP64 peak the pass roofline uses: max(DFMA, DMMA) measured by tools/fp64_peak.cu
    on a B200 of this pool (profiles/r02_fp64_peak.json, 37.0 / 37.1 TF at 1965 MHz)."""
    p = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return max(float(d["dfma_tflops"]), float(d["dmma_tflops"])), \
            "measured (profiles/r02_fp64_peak.json: tools/fp64_peak.cu, DFMA %.1f / DMMA %.1f TF)" % (
                d["dfma_tflops"], d["dmma_tflops"])
    except Exception:
        return F64_NOMINAL_TFLOPS, "nominal B200 datasheet (profiles/r02_fp64_peak.json absent)"
METRIC = "gates/s (circuit time & HBM GB/s reported alongside)"


def load_peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples nvidia-smi clocks and throttle reasons while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuReference:
    """The reference's CPU path — the oracle restatement of run_local (Alg. 3/4 +
    apply_multi), unfused, one pass per gate, on every host thread — on
    the full-size state, built for this host (-O3 -march=native -fcx-limited-range,
    BASELINE.md §3).  The circuit comes from the restated generators with the reference's
    own gate matrices (oracle/gen.cpp + oracle/_ref), so this leg never loads the product
    libraries.  The state is allocated and first-touched once, by the worker pool; every
    timed call runs gates in place (no state copy, no export inside the timer)."""

    def __init__(self, spec: str):
        from oracle import pyoracle

        self.po = pyoracle
        self.lib = pyoracle.native_lib()
        self.circ = pyoracle.generate(spec)
        self.spec = spec
        self.n = self.circ.n
        self.threads = int(self.lib.orc_default_threads())
        self.amps = np.empty(1 << self.n, dtype=np.complex128)
        self.lib.orc_fill_basis(self.n, self.amps.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(0),
                                self.threads)
        self.next_gate = 0
        self.by_class: dict = {}

    def _class(self, i: int) -> str:
        r = self.circ.recs[i]
        return "cx" if r.nctrl else "1q"

    def run(self, budget_s: float, min_gates: int = 1) -> dict:
        """Runs consecutive gates (wrapping to |0> after the last) until budget_s of CPU
        time and at least min_gates; each gate is timed alone."""
        done, secs, moved = 0, 0.0, 0.0
        N = 1 << self.n
        while secs < budget_s or done < min_gates:
            if self.next_gate >= self.circ.nr:
                self.lib.orc_fill_basis(self.n, self.amps.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(0),
                                        self.threads)
                self.next_gate = 0
            g = self.circ.slice(self.next_gate, self.next_gate + 1)
            t0 = time.perf_counter()
            self.po.run_local(g, self.amps, self.threads, inplace=True, library=self.lib)
            dt = time.perf_counter() - t0
            cls = self._class(self.next_gate)
            # algorithmic bytes: a 1q gate streams the state once (r+w); CX touches the half with control = 1
            b = 32.0 * N * (0.5 if cls == "cx" else 1.0)
            c = self.by_class.setdefault(cls, {"gates": 0, "seconds": 0.0, "bytes": 0.0})
            c["gates"] += 1
            c["seconds"] += dt
            c["bytes"] += b
            moved += b
            secs += dt
            done += 1
            self.next_gate += 1
        return {"gates": done, "seconds": secs, "bytes": moved}

    def summary(self, gates: int, secs: float, moved: float) -> dict:
        classes = {k: {"gates": v["gates"], "ms_per_gate": 1e3 * v["seconds"] / v["gates"],
                       "gbs": v["bytes"] / v["seconds"] / 1e9}
                   for k, v in self.by_class.items() if v["gates"]}
        return {"value": gates / secs if secs > 0 else 0.0, "unit": "gates/s", "cores": self.threads,
                "kind": "port", "gates": gates, "seconds": secs, "gbs": moved / secs / 1e9 if secs else None,
                "per_class": classes, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                "oracle_build": "g++ -O3 -march=native -fcx-limited-range (built on this host)",
                "sample": f"{gates} consecutive gates of {self.spec} at full size (2^{self.n} amplitudes, "
                          f"in place, state first-touched once), oracle run_local (Alg. 3/4, one pass per "
                          f"gate, unfused) on {self.threads} host threads, each gate timed alone"}


def cpu_reference_sample(spec: str, budget_s: float, min_gates: int = 1) -> dict:
    ref = CpuReference(spec)
    r = ref.run(budget_s, min_gates)
    return ref.summary(r["gates"], r["seconds"], r["bytes"])


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    spec = args.workload
    ref = CpuReference(spec)
    # one step = the next bounded slice of the same circuit, in place (the state carries
    # over, as in one long run); warm-up steps are untimed
    for _ in range(args.warmup):
        ref.run(args.ref_budget / 4, 1)
    ref.by_class.clear()
    gates = secs = moved = 0.0
    for _ in range(args.steps):
        r = ref.run(args.ref_budget, 1)
        gates += r["gates"]
        secs += r["seconds"]
        moved += r["bytes"]
    summ = ref.summary(int(gates), secs, moved)
    val = summ["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "gates/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (seeded generator circuits)",
        "config": {"workload": spec, "qubits": ref.n, "ranks": 1},
        "cpu_baseline": {k: summ[k] for k in ("value", "unit", "cores", "kind", "sample", "gbs", "per_class",
                                              "cpu_model", "nproc", "oracle_build")},
        "e2e": {"value": val, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit_json(line)


def e2e_stream(args, pkg, qsv, eng, circ, opts, n_local, gates, rank, world, local, barrier, dist):
    """End-to-end through the public engine API with host buffers: every step uploads
    its input state from pinned host memory, runs the circuit and downloads the final
    state.  Up to three engines (three HBM states, three streams) take steps in turn and
    are staggered with stream events so that uploads follow uploads, runs follow runs and
    downloads follow downloads: in steady state the H2D of step k+1, the run of step k and
    the D2H of step k-1 proceed together (full-duplex PCIe), the way a serving loop would
    stream circuits.  Falls back to fewer engines when states do not fit (one engine =
    strictly sequential copies)."""
    N = 1 << n_local
    L = pkg.load_qsim()
    want = 1 if args.e2e_sequential else max(1, args.e2e_engines)
    engines = [eng]
    while len(engines) < want:
        try:
            cid = None
            if world > 1:
                import torch.distributed as tdist

                obj = [pkg.Engine.comm_unique_id() if rank == 0 else None]
                tdist.broadcast_object_list(obj, src=0)
                cid = obj[0]
            engines.append(pkg.Engine(circ, opts, device=local if world > 1 else 0, rank=rank, nranks=world,
                                      comm_id=cid))
        except Exception as exc:  # no room for another 2^n state
            print(f"bench: e2e uses {len(engines)} engine(s) ({exc})", file=sys.stderr)
            break
    ne = len(engines)
    bufs = [C.c_void_p() for _ in range(1 + ne)]
    for h in bufs:
        if qsv.qsv_host_alloc(C.c_size_t(16 * N), C.byref(h)) != 0:
            for g in bufs:
                if g.value:
                    qsv.qsv_host_free(g)
            for e in engines[1:]:
                e.close()
            return None
    src = np.ctypeslib.as_array(C.cast(bufs[0], C.POINTER(C.c_double)), shape=(2 * N,))
    src[:] = 0.0
    if rank == 0:
        src[0] = 1.0  # |0...0>: the host-side input of every step
    din = C.cast(bufs[0], C.POINTER(C.c_double))
    douts = [C.cast(bufs[1 + i], C.POINTER(C.c_double)) for i in range(ne)]
    streams = [C.c_void_p(e.stream) for e in engines]
    evs = {}

    def event(kind, k):
        ev = C.c_void_p()
        qsv.qsv_event_create(C.byref(ev))
        evs[(kind, k)] = ev
        return ev

    def step(k):
        i = k % ne
        e, s = engines[i], streams[i]
        if ne > 1 and ("up", k - 1) in evs:
            qsv.qsv_stream_wait_event(s, evs[("up", k - 1)])
        L.qsim_engine_upload(e._h, din, C.c_uint64(0), C.c_uint64(N))
        if ne > 1:
            qsv.qsv_event_record(event("up", k), s)
            if ("run", k - 1) in evs:
                qsv.qsv_stream_wait_event(s, evs[("run", k - 1)])
        e.run()
        if ne == 1:
            L.qsim_engine_download(e._h, douts[0], C.c_uint64(0), C.c_uint64(N))
            return
        qsv.qsv_event_record(event("run", k), s)
        if ("down", k - 1) in evs:
            qsv.qsv_stream_wait_event(s, evs[("down", k - 1)])
        L.qsim_engine_download_async(e._h, douts[i], C.c_uint64(0), C.c_uint64(N))
        qsv.qsv_event_record(event("down", k), s)

    def drain():
        for e in engines:
            e.sync()
        for ev in evs.values():
            qsv.qsv_event_destroy(ev)
        evs.clear()

    for k in range(ne):  # warm-up: each engine once (graph capture, attributes)
        step(k)
    drain()
    barrier()
    # the stream of circuits runs `e2e_steps` steps (default max(K, 16)): with three engines in
    # flight, K = 3 would time mostly the pipeline's fill and drain, not its steady state
    nsteps = args.e2e_steps or max(args.steps, 16)
    t0 = time.perf_counter()
    for k in range(nsteps):
        step(k)
    drain()
    e2e_s = (time.perf_counter() - t0) / nsteps
    if dist is not None:
        import torch

        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # the result of the last step is on the host: check it is a normalised state
    last = np.ctypeslib.as_array(C.cast(bufs[1 + (nsteps - 1) % ne], C.POINTER(C.c_double)), shape=(2 * N,))
    local_norm = float(np.dot(last, last))
    for e in engines[1:]:
        e.close()
    for h in bufs:
        qsv.qsv_host_free(h)
    api = (f"qsim_engine_upload -> qsim_engine_run -> qsim_engine_download_async on {ne} engines, staggered by "
           "stream events (H2D(k+1) | run(k) | D2H(k-1)); pinned host buffers, full state in and out"
           if ne > 1 else
           "qsim_engine_upload -> qsim_engine_run -> qsim_engine_download (pinned host buffers, full state in and out)")
    out = {"value": gates / e2e_s, "unit": "gates/s", "steps": nsteps, "h2d_bytes_per_step": 16 * N * world,
           "d2h_bytes_per_step": 16 * N * world, "seconds_per_step": e2e_s, "engines": ne,
           "host_norm_rank_shard": local_norm, "api": api}
    # the bound at N = 1: this GPU's PCIe with both directions busy (tools/pcie_probe.py on this
    # pool); with N > 1 the GPUs share the host's memory and root complexes, which the probe of
    # one link does not bound, so no roofline is claimed there
    try:
        if world != 1:
            raise ValueError("multi-GPU")
        with open(os.path.join(ROOT, "profiles", "r02_pcie_probe.json")) as f:
            duplex = float(json.load(f)["duplex_total_gbs"])
        floor_s = 2 * 16 * N / (duplex * 1e9)  # per GPU: its shard in and out over its own link
        out["pcie_roofline"] = {"duplex_gbs_measured": duplex, "floor_s_per_step": floor_s,
                                "frac": floor_s / e2e_s, "source": "profiles/r02_pcie_probe.json"}
    except (OSError, KeyError, ValueError):
        pass
    return out


# Native libraries (NCCL's version banner, CUDA warnings) may write to fd 1; the
# contract is ONE JSON line on stdout, so fd 1 points at stderr until emit_json.
_STDOUT_FD = None


def quiet_stdout():
    global _STDOUT_FD
    if _STDOUT_FD is None:
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)


def emit_json(line):
    sys.stdout.flush()
    if _STDOUT_FD is not None:
        os.dup2(_STDOUT_FD, 1)
    print(json.dumps(line), flush=True)


EXTRA_CONFIGS = [
    # (label, spec, PlanOptions overrides): BASELINE.json configs[0], [1] contraction off, [2], [3]
    ("qft24", "qft:24", {}),
    ("random30_fusion_off", "random:30:20:2", {"fusion": False}),
    ("uccsd28", "uccsd:28:100000:3", {}),
    ("hea33", "hea:33:5:4", {}),
]


def measure_config(pkg, spec, overrides, steps, hbm_peak, f64_peak, device=0) -> dict:
    """One BASELINE.json config on one GPU: plan + JIT (untimed), 1 warm-up run, then `steps`
    timed runs from |0...0> (CUDA events on the engine stream, clocks sampled), plus the
    per-pass profile for the roofline fraction.  The engine is freed before returning."""
    opts = pkg.PlanOptions()
    for k, v in overrides.items():
        setattr(opts, k, v)
    circ = pkg.Circuit.generate(spec)
    t0 = time.perf_counter()
    eng = pkg.Engine(circ, opts, device=device)
    setup_s = time.perf_counter() - t0
    jit = eng.jit_info()
    st = eng.stats
    info = eng.steps()
    eng.set_basis(0)
    eng.run()
    eng.sync()
    clocks = ClockSampler(device)
    clocks.start()
    ms = eng.time(steps, basis=0) / steps
    clk = clocks.stop()
    eng.set_basis(0)
    prof = eng.profile()
    norm = eng.norm_sq()
    eng.close()
    pass_ms = [p for p, s in zip(prof, info) if s["kind"] == "pass"]
    pbytes = [s["hbm_bytes"] for s in info if s["kind"] == "pass"]
    pflops = [s["flops"] for s in info if s["kind"] == "pass"]
    t_roof = sum(max(b / (hbm_peak * 1e9), f / (f64_peak * 1e12)) for b, f in zip(pbytes, pflops))
    per_pass_frac = [max(b / (hbm_peak * 1e9), f / (f64_peak * 1e12)) / (t / 1e3)
                     for b, f, t in zip(pbytes, pflops, pass_ms) if t > 0]
    return {
        "workload": spec, "options": overrides or "default", "gates": st["gates_in"], "passes": st["passes"],
        "circuit_time_s": ms / 1e3, "gates_per_s": st["gates_in"] / (ms / 1e3), "timed_runs": steps,
        "hbm_gbs_avg": (sum(pbytes) / 1e9) / (sum(pass_ms) / 1e3) if pass_ms else None,
        "hbm_floor_s": sum(pbytes) / (hbm_peak * 1e9),
        "roofline_time_s": t_roof, "roofline_frac": t_roof / (ms / 1e3),
        "passes_at_or_above_0.70": sum(1 for f in per_pass_frac if f >= 0.70),
        "min_pass_frac": min(per_pass_frac) if per_pass_frac else None,
        "achieved_tflops": sum(pflops) / (sum(pass_ms) / 1e3) / 1e12 if pass_ms else None,
        "norm_error": abs(norm - 1.0), "jit_kernels": jit["kernels"], "setup_s": round(setup_s, 2),
        "clocks": clk,
    }


def main():
    quiet_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="random:30:20:2")
    ap.add_argument("--fusion", default="on", choices=["on", "off"])
    ap.add_argument("--tile-k", type=int, default=None)
    ap.add_argument("--budget", type=float, default=None)
    ap.add_argument("--relabel", type=int, default=1, choices=[0, 1, 2],
                    help="tile-qubit relabelling: 0 off, 1 auto (kept when it saves passes), 2 always")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true",
                    help="skip the other BASELINE.json configs (QFT-24, random-30 DAGC off, UCCSD-28, HEA-33)")
    ap.add_argument("--e2e-sequential", action="store_true", help="one engine, no copy/compute overlap")
    ap.add_argument("--e2e-steps", type=int, default=0, help="steps of the e2e stream (default max(K, 16))")
    ap.add_argument("--e2e-engines", type=int, default=3, help="engines (HBM states) the e2e stream rotates over")
    ap.add_argument("--ref-budget", type=float, default=12.0, help="seconds of CPU work per reference step")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds for the cpu_baseline sample")
    ap.add_argument("--cpu-min-gates", type=int, default=45, help="gates the cpu_baseline sample covers at least")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 untimed warm-up steps

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import paper_2509_04955_b200 as pkg

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    dist = None
    comm_id = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
        obj = [pkg.Engine.comm_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        comm_id = obj[0]

    opts = pkg.PlanOptions()
    opts.fusion = args.fusion == "on"
    if args.tile_k:
        opts.tile_k = args.tile_k
    if args.budget:
        opts.pass_budget = args.budget
    opts.relabel = args.relabel
    circ = pkg.Circuit.generate(args.workload)
    n = circ.n
    t_plan0 = time.perf_counter()
    eng = pkg.Engine(circ, opts, device=local if world > 1 else 0, rank=rank, nranks=world, comm_id=comm_id)
    jit = eng.jit_info()
    if opts.jit and jit["kernels"] == 0:
        print("bench: WARNING specialised (NVRTC) pass kernels unavailable; interpreter kernel in use",
              file=sys.stderr)
    plan_s = time.perf_counter() - t_plan0
    st = eng.stats
    steps_info = eng.steps()
    n_local = eng.n_local

    def barrier():
        if dist is not None:
            dist.barrier()

    def one_step():
        eng.set_basis(0)
        eng.run()

    # warm-up (also captures the CUDA graph of the program)
    for _ in range(args.warmup):
        one_step()
    eng.sync()

    # timed region: CUDA events on the engine stream bracket exactly K steps
    import ctypes as C

    qsv = pkg.load_qsv()
    clocks = ClockSampler(local if world > 1 else 0)
    ev = [C.c_void_p(), C.c_void_p()]
    barrier()
    eng.sync()
    clocks.start()
    t0 = time.perf_counter()
    # qsv_program_time records one CUDA event before and one after the K steps on
    # the engine stream; each step = reset to |0...0> (memset + 1 kernel) + program
    ms_total = eng.time(args.steps, basis=0)
    eng.sync()
    wall = time.perf_counter() - t0
    barrier()
    clk = clocks.stop()
    ms_step = ms_total / args.steps
    if dist is not None:
        import torch

        t = torch.tensor([ms_step], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    gates = st["gates_in"]
    value = gates / (ms_step / 1e3)

    # per-step device profile (separate run; CUDA events per pass on the engine stream)
    eng.set_basis(0)
    prof = eng.profile()
    pass_ms = [p for p, s in zip(prof, steps_info) if s["kind"] == "pass"]
    # swaps the timed runs actually move: the leading ones act on the basis start |0...0> and
    # become an index relabel (QSV_BASIS_SWAPS, default on; the profile run still moves them)
    lead = 0
    if os.environ.get("QSV_BASIS_SWAPS", "1") != "0":
        while lead < len(steps_info) and steps_info[lead]["kind"] == "swap":
            lead += 1
    swap_ms = [p for i, (p, s) in enumerate(zip(prof, steps_info)) if s["kind"] == "swap" and i >= lead]
    pass_bytes = [s["hbm_bytes"] for s in steps_info if s["kind"] == "pass"]
    pass_flops = [s["flops"] for s in steps_info if s["kind"] == "pass"]
    hbm_peak, hbm_src = load_peaks()
    f64_peak, f64_src = load_f64_peak()
    avg_pass_ms = sum(pass_ms) / max(len(pass_ms), 1)
    achieved = (sum(pass_bytes) / max(len(pass_bytes), 1)) / (avg_pass_ms / 1e3) / 1e9 if pass_ms else 0.0
    t_roof = sum(max(b / (hbm_peak * 1e9), f / (f64_peak * 1e12)) for b, f in zip(pass_bytes, pass_flops))
    nvl = sum(s["nvl_bytes"] for s in steps_info)
    t_roof += nvl / 770e9
    norm = eng.norm_sq()  # this rank's shard; summed over the ranks below (a whole-state check at every N)
    if dist is not None:
        import torch

        tn = torch.tensor([norm], dtype=torch.float64, device="cuda")
        dist.all_reduce(tn, op=dist.ReduceOp.SUM)
        norm = float(tn.item())

    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("workload") == args.workload:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # e2e: the same circuit through the public engine API with pinned host buffers:
    # H2D of the initial state, the run, D2H of the final state, every step.
    e2e = None
    if not args.no_e2e:
        e2e = e2e_stream(args, pkg, qsv, eng, circ, opts, n_local, gates, rank, world, local, barrier, dist)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_sample(args.workload, budget_s=args.cpu_budget, min_gates=args.cpu_min_gates)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "gbs", "per_class", "cpu_model",
                                   "nproc", "oracle_build")}

    extra = None
    if rank == 0 and world == 1 and not args.no_extra_configs:
        eng.close()  # HEA-33 needs 128 GiB of the GPU
        extra = {}
        for label, spec, ov in EXTRA_CONFIGS:
            try:
                extra[label] = measure_config(pkg, spec, ov, 2, hbm_peak, f64_peak)
            except Exception as ex:  # reported, never silently dropped
                extra[label] = {"workload": spec, "error": str(ex)[:300]}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    launches = (len(pass_ms) + 1) * args.steps  # pass kernels + the basis-set kernel
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "gates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c128 (f64)",
        "data": "synthetic (seeded generator circuit, state from |0...0>)",
        "config": {
            "workload": args.workload, "qubits": n, "local_qubits": n_local, "ranks": world,
            "fusion": args.fusion, "tile_k": opts.tile_k, "pass_budget": opts.pass_budget,
            "relabel": args.relabel, "jit_kernels": jit["kernels"], "jit_seconds": round(jit["seconds"], 2),
            "gates": gates, "ops_after_fusion": st["ops_fused"], "ops_final": st["ops_final"],
            "passes": st["passes"], "swaps": st["swaps"], "swaps_relabelled_on_basis_start": lead,
            "plan_seconds": plan_s,
            "l2": "state (16 B x 2^n) >> 126 MB L2; no flush needed",
        },
        "circuit_time_s": ms_step / 1e3,
        "hbm_gbs_avg": (sum(pass_bytes) / 1e9) / (sum(pass_ms) / 1e3) if pass_ms else None,
        "roofline": {
            "bound": "hbm", "kernel": "qsv_jit_* (NVRTC-specialised fused multi-op pass kernels; qsv::pass_kernel is the interpreter fallback)",
            "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak if hbm_peak else None, "traffic": traffic,
            "peak_source": hbm_src,
            "algorithmic_bytes_per_launch": sum(pass_bytes) / max(len(pass_bytes), 1),
            "avg_launch_ms": avg_pass_ms,
            "circuit_roofline_time_s": t_roof, "circuit_roofline_frac": t_roof / (ms_step / 1e3),
            "f64_peak_tflops": f64_peak, "f64_peak_source": f64_src,
            "achieved_tflops": sum(pass_flops) / (sum(pass_ms) / 1e3) / 1e12 if pass_ms else None,
        },
        "swap_ms_total": sum(swap_ms) if swap_ms else 0.0,
        # BBOP: (step time - local passes alone) / swaps alone, both from the per-step profile
        "swap_exposed_frac": ((ms_step - sum(pass_ms)) / sum(swap_ms)) if swap_ms and sum(swap_ms) > 0 else None,
        "norm_error": abs(norm - 1.0),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "configs": extra,
        "gpu_launches": launches,
        "clocks": clk,
        "wall_s_timed_region": wall,
    }
    emit_json(line)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
