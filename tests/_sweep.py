import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg
specs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["random:30:20:2", "hea:30:5:4", "qft:30"]
grid = [dict(), dict(min_low=4), dict(min_low=3), dict(pass_budget=128), dict(min_low=4, pass_budget=128), dict(min_low=3, pass_budget=128), dict(tile_k=10), dict(tile_k=10, min_low=4, pass_budget=128)]
for spec in specs:
    c = pkg.Circuit.generate(spec)
    for kw in grid:
        o = pkg.PlanOptions(**kw)
        e = pkg.Engine(c, o)
        e.set_basis(0); e.run(); e.sync()
        t = e.time(3) / 3
        print(spec, kw, "ms %.1f" % t, "passes", e.stats["passes"], e.jit_info(), flush=True)
        e.close()
