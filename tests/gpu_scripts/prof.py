import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg
spec = sys.argv[1] if len(sys.argv) > 1 else "random:28:20:2"
c = pkg.Circuit.generate(spec)
e = pkg.Engine(c, pkg.PlanOptions())
e.set_basis(0)
prof = e.profile()
st = e.steps()
for i, (p, s) in enumerate(zip(prof, st)):
    if i < 200:
        print(i, "%.3f ms" % p, s["nops"], "%.1f GB/s" % (s["hbm_bytes"] / p / 1e6),
              "%.2f TF" % (s.get("flops", 0) / p / 1e9), "%.0f flop/amp" % (s.get("flops", 0) / (s["hbm_bytes"] / 32)))
print("total", sum(prof))
