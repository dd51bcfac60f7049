"""Per-pass JIT vs interpreter times: args spec [spec ...].  Prints one JSON line per spec with
the two circuit times, the JIT compile time and a histogram of per-pass interp/JIT ratios by
op count, so a JIT policy (which passes are worth compiling) can be read off."""
import json
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg  # noqa: E402

for spec in sys.argv[1:]:
    c = pkg.Circuit.generate(spec)
    res = {"spec": spec}
    prof = {}
    for jit in (1, 0):
        t0 = time.time()
        e = pkg.Engine(c, pkg.PlanOptions(jit=bool(jit)))
        res[f"setup_s_jit{jit}"] = round(time.time() - t0, 2)
        e.time(1, 0)
        res[f"ms_jit{jit}"] = round(e.time(3, 0) / 3, 2)
        e.set_basis(0)
        prof[jit] = e.profile()
        steps = e.steps()
        if jit:
            res["jit"] = e.jit_info()
        e.close()
    buckets = {}
    for s, a, b in zip(steps, prof[1], prof[0]):
        if s["kind"] != "pass":
            continue
        key = min(s["nops"], 32)
        bk = buckets.setdefault(key, [0, 0.0, 0.0])
        bk[0] += 1
        bk[1] += a
        bk[2] += b
    res["by_nops"] = {k: {"passes": v[0], "jit_ms": round(v[1], 2), "interp_ms": round(v[2], 2)}
                      for k, v in sorted(buckets.items())}
    print(json.dumps(res), flush=True)
