"""Runs one circuit on N GPUs (one Engine per GPU, one host thread each) with the
PipelineTrace on and writes rank 0's trace as JSON:
  python tools/trace_run.py <spec> <ngpus> <out.json>   (env: QSV_OVERLAP, QSV_SWAP_MODE, ...)
"""
import json
import os
import sys
import threading

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
import paper_2509_04955_b200 as pkg  # noqa: E402


def main():
    spec, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    c = pkg.Circuit.generate(spec)
    cid = pkg.Engine.comm_unique_id()
    engines = [None] * n

    def make(r):
        engines[r] = pkg.Engine(c, pkg.PlanOptions(), device=r, rank=r, nranks=n, comm_id=cid)

    def each(fn):
        th = [threading.Thread(target=fn, args=(e,)) for e in engines]
        [t.start() for t in th]
        [t.join() for t in th]

    th = [threading.Thread(target=make, args=(r,)) for r in range(n)]
    [t.start() for t in th]
    [t.join() for t in th]

    def warm(e):
        e.set_basis(0)
        e.run()
        e.sync()

    def traced(e):
        e.trace_enable(True)
        e.set_basis(0)
        e.run()
        e.sync()

    each(warm)
    each(traced)
    tr = engines[0].trace()
    steps = engines[0].steps()
    total = max(r["end_ms"] for r in tr) - min(r["start_ms"] for r in tr)
    json.dump({"spec": spec, "ngpus": n, "env": {k: v for k, v in os.environ.items() if k.startswith("QSV_")},
               "total_ms": total, "steps": steps, "trace": tr}, open(out, "w"))
    busy = {}
    for r in tr:
        busy.setdefault(r["kind"], 0.0)
        busy[r["kind"]] += r["end_ms"] - r["start_ms"]
    print(spec, n, "total %.1f ms" % total, {k: round(v, 1) for k, v in busy.items()})
    for e in engines:
        e.close()


if __name__ == "__main__":
    main()
