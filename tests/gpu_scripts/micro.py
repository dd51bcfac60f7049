import sys, os, math
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np
import paper_2509_04955_b200 as pkg
n = 30
def block_circ(qs, layers, cx=True):
    c = pkg.Circuit.empty(n)
    for l in range(layers):
        for i, q in enumerate(qs):
            c.add("rx" if (l + i) % 2 else "ry", [q], [0.1 + 0.01 * l + 0.001 * i])
        if cx:
            if l % 2 == 0:
                c.add("cx", [qs[0], qs[1]]); c.add("cx", [qs[2], qs[3]]) if len(qs) > 3 else None
            else:
                c.add("cx", [qs[1], qs[2]])
    return c
def timeit(c, opts, reps=3):
    e = pkg.Engine(c, opts)
    e.set_basis(0); e.run(); e.sync()
    ms = e.time(reps) / reps
    st = e.stats
    e.close()
    return ms, st
big = pkg.PlanOptions(pass_budget=1e9, tile_k=11, rblock_k=4)
c0 = pkg.Circuit.empty(n).add("rz", [5], [0.3])
ms, st = timeit(c0, big)
print("one diag op pass: %.3f ms (%.0f GB/s)" % (ms, 32 * 2**n / ms / 1e6), st["passes"])
for qs in ([0, 1, 2, 3], [4, 5, 6, 7], [20, 21, 22, 23], [1, 8, 15, 25]):
    for layers in (1, 2, 4, 8, 16):
        c = block_circ(qs, layers)
        ms, st = timeit(c, big)
        print("RB4 qs=%s layers=%2d prims~%3d ops=%d passes=%d: %.3f ms" % (qs, layers, layers * 4 + (layers * 3 + 1) // 2, st["ops_final"], st["passes"], ms), flush=True)
for qs in ([0, 1, 2], [20, 21, 22]):
    for layers in (1, 4, 16):
        c = block_circ(qs, layers, cx=False)
        ms, st = timeit(c, pkg.PlanOptions(pass_budget=1e9, tile_k=10, rblock_k=3))
        print("RB3 qs=%s layers=%2d ops=%d passes=%d: %.3f ms" % (qs, layers, st["ops_final"], st["passes"], ms), flush=True)
# dense ops (no register blocks): k=1 gates on distinct qubits, one pass
for k in (1, 2, 3, 4):
    rng = np.random.default_rng(k)
    for nops in (1, 4, 8):
        c = pkg.Circuit.empty(n)
        for i in range(nops):
            q, r = np.linalg.qr(rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k)))
            c.add_unitary(q, [ (i * k + j) % 10 + (20 if j % 2 else 0) for j in range(k)] if k > 1 else [i % 10])
        ms, st = timeit(c, pkg.PlanOptions(pass_budget=1e9, tile_k=11, register_blocks=False, fuse_k=1))
        print("DENSE k=%d nops=%d passes=%d: %.3f ms" % (k, nops, st["passes"], ms), flush=True)
for nops in (1, 4, 8, 16):
    c = pkg.Circuit.empty(n)
    for i in range(nops):
        c.add("rz", [i], [0.1 * i + 0.05])
        c.add("cp", [i + 10, 29 - i], [0.2])
    ms, st = timeit(c, pkg.PlanOptions(pass_budget=1e9, tile_k=11, register_blocks=False))
    print("DIAG/PHASE nops=%d ops=%d passes=%d: %.3f ms" % (nops, st["ops_final"], st["passes"], ms), flush=True)
