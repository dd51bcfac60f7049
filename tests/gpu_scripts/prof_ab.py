"""A/B timing of plan options: args spec, then k=v option sets separated by '/'."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg
spec = sys.argv[1]
c = pkg.Circuit.generate(spec)
for oset in sys.argv[2:]:
    kw = {}
    for kv in oset.split(","):
        if kv:
            k, v = kv.split("=")
            kw[k] = float(v) if "." in v else int(v)
    e = pkg.Engine(c, pkg.PlanOptions(**kw))
    e.time(1, 0)
    ms = e.time(3, 0) / 3
    print(spec, oset or "default", os.environ.get("QSV_PLAN_FIXED_L", ""), "passes", len(e.steps()), "ms/iter %.1f" % ms,
          "jit", e.jit_info()["kernels"], flush=True)
    e.close()
