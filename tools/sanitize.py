"""Small circuits through every pass-kernel flavour: the NVRTC-specialised kernels, the
interpreter, relabel passes and relabels folded into register-block stores, dense k<=5
ops and 12-qubit tiles.  Each result is checked against the CPU oracle and its bitwise
digest printed, so runs under the debug switches (QSV_DEBUG_POISON=1: NaN-filled tile
buffers before every TMA load; QSV_DEBUG_GRID=N: N persistent CTAs, another tile order
and pipeline phase) can be compared bit for bit (tests/test_gpu_parity.py).  Also the
compute-sanitizer driver where that tool is available:
  compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.join(os.path.dirname(__file__), "..")))
import numpy as np  # noqa: E402

import paper_2509_04955_b200 as pkg  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

CASES = [
    ("random:13:6:2", dict()),                                   # JIT, register blocks, epilogues
    ("uccsd:12:200:3", dict(relabel=2)),                         # relabel ops + folded relabel stores
    ("qft:12", dict()),                                          # PHASEPROD / diagonal epilogues
    ("random:12:6:2", dict(jit=False, relabel=2, tile_k=8, min_low=4)),  # interpreter + relabel
    ("random:12:5:2", dict(register_blocks=False, fuse_k=4, tile_k=10)),  # dense k = 4 ops
    ("random:12:5:2", dict(register_blocks=False, fuse_k=5, pass_budget=500)),  # dense k = 5
    ("random:13:6:2", dict(tile_k=12, relabel=2)),               # 12-qubit tiles (256 threads)
]


def main():
    worst = 0.0
    for spec, kw in CASES:
        c = pkg.Circuit.generate(spec)
        e = pkg.Engine(c, pkg.PlanOptions(**kw))
        e.set_basis(0)
        e.run()
        e.sync()
        got = e.download()
        dig = e.digest()
        e.close()
        err = float(np.abs(got - O.run_local(c)).max())
        worst = max(worst, err)
        print(f"DIGEST {spec} {sorted(kw.items())} {dig:016x}", flush=True)
        print(f"{spec} {kw} max-abs {err:.2e}", flush=True)
    assert worst <= 1e-10, worst
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
