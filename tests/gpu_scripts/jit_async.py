"""Cold-start latency of the specialised kernels: time to the first result with the synchronous
compile (PlanOptions(jit=1)) and with the background compile (jit=2, interpreted runs until the
kernels load), each from an empty JIT cache.  Args: spec [spec ...].  One JSON line per spec."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg  # noqa: E402


def first_result(c, jit):
    os.environ["QSV_JIT_CACHE"] = tempfile.mkdtemp(prefix=f"qsv_jit_cold{jit}_")
    t0 = time.time()
    e = pkg.Engine(c, pkg.PlanOptions(jit=jit))
    t_create = time.time() - t0
    e.set_basis(0)
    e.run()
    e.sync()
    t_first = time.time() - t0
    runs = 1
    if jit == 2:  # keep producing results until the kernels are in
        while e.jit_info()["kernels"] == 0:
            e.set_basis(0)
            e.run()
            e.sync()
            runs += 1
    t_switch = time.time() - t0
    e.jit_wait()
    e.set_basis(0)
    e.run()
    e.sync()
    ms_after = e.time(2, 0) / 2
    info = e.jit_info()
    e.close()
    return {"create_s": round(t_create, 2), "first_result_s": round(t_first, 2), "runs_before_switch": runs,
            "switch_s": round(t_switch, 2), "ms_per_run_after": round(ms_after, 1), "kernels": info["kernels"],
            "compile_s": round(info["seconds"], 1)}


for spec in sys.argv[1:]:
    c = pkg.Circuit.generate(spec)
    print(json.dumps({"spec": spec, "sync": first_result(c, 1), "async": first_result(c, 2)}), flush=True)
