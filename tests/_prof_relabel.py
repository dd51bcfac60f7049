import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg
from tests import dist_emulator as E
spec = sys.argv[1] if len(sys.argv) > 1 else "random:30:20:2"
c = pkg.Circuit.generate(spec)
for rl in (0, 2):
    o = pkg.PlanOptions(relabel=rl)
    steps, *_ = E.export_plan(c, o, c.n)
    e = pkg.Engine(c, o)
    e.set_basis(0)
    prof = e.profile()
    prof = e.profile()
    st = e.steps()
    tot = 0
    for i, (p, s, d) in enumerate(zip(prof, st, steps)):
        tot += p
        print(rl, i, "%.3f ms" % p, s["nops"], d.has_relabel, "%.0f GB/s" % (s["hbm_bytes"] / p / 1e6))
    print("relabel", rl, "total", tot, "jit", e.jit_info())
    e.close()
