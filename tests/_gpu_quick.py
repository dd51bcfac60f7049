import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np
import paper_2509_04955_b200 as pkg
from oracle import pyoracle as O
rng = np.random.default_rng(0)
def rand_state(n):
    a = rng.normal(size=1<<n) + 1j*rng.normal(size=1<<n); return a/np.linalg.norm(a)
bad = 0
for spec in ["qft:5", "random:8:4:2", "random:12:8:2", "hea:12:3:4", "qft:14", "random:16:10:2", "uccsd:14:400:3", "qaoa:13:2:1", "qft:18"]:
    c = pkg.Circuit.generate(spec)
    n = c.n
    a = rand_state(n)
    ref = O.run_local(c, a)
    for opts in [pkg.PlanOptions(), pkg.PlanOptions(jit=False), pkg.PlanOptions(fusion=False, multi_op_passes=False), pkg.PlanOptions(register_blocks=False, fuse_k=4, tile_k=10), pkg.PlanOptions(fuse_k=5, tile_k=11, pass_budget=400, register_blocks=False), pkg.PlanOptions(rblock_k=3, tile_k=10)]:
        e = pkg.Engine(c, opts)
        e.upload(a); e.run(); e.sync()
        got = e.download()
        err = np.abs(got-ref).max()
        bad += err > 1e-10
        if err > 1e-10: print("BAD", spec, opts, err)
        e.close()
print("BAD", bad, flush=True)
for spec in ["random:30:20:2", "qft:30", "hea:30:5:4"]:
    c = pkg.Circuit.generate(spec)
    for opts in [pkg.PlanOptions(jit=False), pkg.PlanOptions(), pkg.PlanOptions(pass_budget=96), pkg.PlanOptions(pass_budget=128), pkg.PlanOptions(pass_budget=160)]:
        e = pkg.Engine(c, opts)
        e.set_basis(0); e.run(); e.sync()
        t = e.time(2)/2
        st = e.steps()
        hb = sum(s["hbm_bytes"] for s in st)
        fl = sum(s["flops"] for s in st)
        prof = e.profile()
        print(spec, "jit" if opts.jit else "interp", e.jit_info(), opts.pass_budget, "ms %.1f" % t, "passes", e.stats["passes"], "ops", e.stats["ops_final"], "GB/s %.0f" % (hb/t/1e6), "TF %.2f" % (fl/t/1e9), "min-pass %.2f max %.2f" % (min(prof), max(prof)), flush=True)
        e.close()
