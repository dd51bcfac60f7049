import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2509_04955_b200 as pkg
spec = sys.argv[1] if len(sys.argv) > 1 else "random:28:20:2"
c = pkg.Circuit.generate(spec)
e = pkg.Engine(c, pkg.PlanOptions())
e.set_basis(0)
prof = e.profile()
st = e.steps()
# roofline per pass: max(bytes / measured HBM, flops / measured FP64) over its time
import json
try:
    hbm = float(json.load(open(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    hbm = 6553.9
f64 = 37.125
fr = []
for i, (p, s) in enumerate(zip(prof, st)):
    roof = max(s["hbm_bytes"] / (hbm * 1e9), s.get("flops", 0) / (f64 * 1e12)) * 1e3
    if s["kind"] == "pass":
        fr.append(roof / p)
    if i < 200:
        print(i, "%.3f ms" % p, s["nops"], "%.1f GB/s" % (s["hbm_bytes"] / p / 1e6),
              "%.2f TF" % (s.get("flops", 0) / p / 1e9), "%.0f flop/amp" % (s.get("flops", 0) / (s["hbm_bytes"] / 32)),
              "roofline %.3f ms frac %.2f" % (roof, roof / p))
if fr:
    print("passes", len(fr), ">= 0.70:", sum(1 for f in fr if f >= 0.70), "min frac %.2f" % min(fr),
          "mean frac %.2f" % (sum(fr) / len(fr)))
print("total", sum(prof))
