"""TEST INFRASTRUCTURE: numpy emulation of a rank's device program (include/qsv.h
semantics) used to check the multi-rank planner and the swap protocol on CPU
with torch.distributed/gloo.  Never used by the product path."""
import ctypes as C

import numpy as np

import paper_2509_04955_b200 as pkg

QSV_MAX_HIGH = 8


class Step(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tile_k", C.c_int32), ("nhigh", C.c_int32), ("high", C.c_int32 * QSV_MAX_HIGH),
                ("op_begin", C.c_int32), ("op_count", C.c_int32), ("has_relabel", C.c_int32),
                ("relabel", C.c_int32 * 16), ("swap_global", C.c_int32),
                ("swap_local", C.c_int32), ("chunk_log2", C.c_int32), ("nbuf", C.c_int32)]


class Op(C.Structure):
    _fields_ = [("kind", C.c_int32), ("k", C.c_int32), ("qubits", C.c_int32 * 8), ("ctrl_mask", C.c_uint64),
                ("mat_off", C.c_int64), ("prim_begin", C.c_int32), ("nprim", C.c_int32),
                ("qmask", C.c_uint64)]


class Prim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("pad", C.c_int32),
                ("mat_off", C.c_int64)]


def export_plan(circ, opts, n_local):
    L = pkg.load_qsim()
    ns, no, npr, pl = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    o = opts.to_c()
    rc = L.qsim_plan_export(circ._h, C.byref(o), n_local, C.byref(ns), C.byref(no), C.byref(npr), C.byref(pl),
                            None, None, None, None)
    assert rc == 0, L.qsim_last_error()
    steps = (Step * max(ns.value, 1))()
    ops = (Op * max(no.value, 1))()
    prims = (Prim * max(npr.value, 1))()
    pool = np.zeros(max(pl.value, 1), dtype=np.complex128)
    rc = L.qsim_plan_export(circ._h, C.byref(o), n_local, C.byref(ns), C.byref(no), C.byref(npr), C.byref(pl),
                            steps, ops, prims, pool.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)))
    assert rc == 0
    return list(steps)[:ns.value], list(ops)[:no.value], list(prims)[:npr.value], pool


def _groups(l, rank, targets, ctrl_mask, n_local):
    """Local base indices (target bits 0, all control bits 1) of this rank's shard."""
    full = (np.uint64(rank) << np.uint64(n_local)) | np.arange(1 << l, dtype=np.uint64)
    sel = (full & np.uint64(ctrl_mask)) == np.uint64(ctrl_mask)
    for t in targets:
        sel &= ((full >> np.uint64(t)) & np.uint64(1)) == 0
    return np.nonzero(sel)[0].astype(np.int64), full


def _apply_matrix(psi, bases, targets, m):
    d = 1 << len(targets)
    offs = np.zeros(d, dtype=np.int64)
    for j in range(d):
        for i, t in enumerate(targets):
            if j >> i & 1:
                offs[j] |= 1 << t
    idx = bases[:, None] + offs[None, :]
    psi[idx] = psi[idx] @ m.T


def apply_op(psi, op, prims, pool, rank, n_local):
    l = n_local
    kind = op.kind
    if kind in (0, 2):  # DENSE / XPERM
        t = [op.qubits[i] for i in range(op.k)]
        d = 1 << op.k
        m = pool[op.mat_off:op.mat_off + d * d].reshape(d, d) if kind == 0 else np.array([[0, 1], [1, 0]], complex)
        bases, _ = _groups(l, rank, t, op.ctrl_mask, n_local)
        _apply_matrix(psi, bases, t, m)
    elif kind == 1:  # DIAG
        q = [op.qubits[i] for i in range(op.k)]
        bases, full = _groups(l, rank, [], op.ctrl_mask, n_local)
        e = np.zeros(bases.size, dtype=np.int64)
        for i, qq in enumerate(q):
            e |= (((full[bases] >> np.uint64(qq)) & np.uint64(1)).astype(np.int64)) << i
        psi[bases] *= pool[op.mat_off + e]
    elif kind == 5:  # PARPHASE
        bases, full = _groups(l, rank, [], op.ctrl_mask, n_local)
        par = np.zeros(bases.size, dtype=np.int64)
        for q in range(64):
            if op.qmask >> q & 1:
                par ^= ((full[bases] >> np.uint64(q)) & np.uint64(1)).astype(np.int64)
        psi[bases] *= pool[op.mat_off + par]
    elif kind == 4:  # PHASEPROD
        bases, full = _groups(l, rank, [], op.ctrl_mask, n_local)
        w = np.full(bases.size, pool[op.mat_off], dtype=np.complex128)
        for p in prims[op.prim_begin:op.prim_begin + op.nprim]:
            on = ((full[bases] >> np.uint64(p.a)) & np.uint64(1)).astype(bool)
            w[on] *= pool[p.mat_off]
        psi[bases] *= w
    elif kind == 3:  # RBLOCK
        k = op.k
        slots = [op.qubits[i] for i in range(k)]
        bases, _ = _groups(l, rank, slots, op.ctrl_mask, n_local)
        for p in prims[op.prim_begin:op.prim_begin + op.nprim]:
            if p.kind in (0, 5, 6):
                _apply_matrix(psi, _groups(l, rank, [slots[p.a]], op.ctrl_mask, n_local)[0], [slots[p.a]],
                              pool[p.mat_off:p.mat_off + 4].reshape(2, 2))
            elif p.kind == 1:
                tt = [slots[p.a], slots[p.b]]
                _apply_matrix(psi, _groups(l, rank, tt, op.ctrl_mask, n_local)[0], tt,
                              pool[p.mat_off:p.mat_off + 16].reshape(4, 4))
            elif p.kind == 2:
                cm = op.ctrl_mask | (1 << slots[p.a])
                b2, _ = _groups(l, rank, [slots[p.b]], cm, n_local)
                _apply_matrix(psi, b2, [slots[p.b]], np.array([[0, 1], [1, 0]], complex))
            else:
                nd = 1 << k
                tab = pool[p.mat_off:p.mat_off + nd]
                e = np.zeros(bases.size, dtype=np.int64)
                idx_all = bases
                offs = np.zeros(nd, dtype=np.int64)
                for j in range(nd):
                    for i, sq in enumerate(slots):
                        if j >> i & 1:
                            offs[j] |= 1 << sq
                idx = idx_all[:, None] + offs[None, :]
                psi[idx] *= tab[None, :]
    else:
        raise ValueError(f"unknown op kind {kind}")


def relabel(psi, s, n_local):
    """Pass relabel: tile bit i (low run, then high[] in order) moves to tile bit relabel[i]."""
    L = s.tile_k - s.nhigh
    slots = list(range(L)) + [s.high[i] for i in range(s.nhigh)]
    dst_of = {slots[i]: slots[s.relabel[i]] for i in range(len(slots))}
    # numpy axes are most-significant first: axis a <-> physical bit n_local-1-a
    perm_src = list(range(n_local))
    for p, d in dst_of.items():
        perm_src[d] = p
    view = psi.reshape((2,) * n_local)
    out = np.transpose(view, [n_local - 1 - perm_src[n_local - 1 - a] for a in range(n_local)])
    psi[:] = out.reshape(-1)


def run_program(psi, steps, ops, prims, pool, rank, n_local, exchange):
    """exchange(psi, g, v, chunk_log2, nbuf) performs the swap collective."""
    for s in steps:
        if s.kind == 0:
            for op in ops[s.op_begin:s.op_begin + s.op_count]:
                apply_op(psi, op, prims, pool, rank, n_local)
            if s.has_relabel:
                relabel(psi, s, n_local)
        else:
            exchange(psi, s.swap_global, s.swap_local, s.chunk_log2, s.nbuf)
    return psi


def swap_indices(n_local, rank, g, v, chunk_log2):
    """The chunk schedule of swap.cu: local indices (bit v = !a) in chunk order."""
    a = (rank >> (g - n_local)) & 1
    sendbit = a ^ 1
    r = np.arange(1 << (n_local - 1), dtype=np.int64)
    lo = r & ((1 << v) - 1)
    idx = ((r ^ lo) << 1) | (sendbit << v) | lo
    c = 1 << chunk_log2
    return [idx[i:i + c] for i in range(0, idx.size, c)]


def validate(steps, ops, prims, pool, n_total, n_local, rank):
    """qsv_program_validate (host-side compile of every pass) on an exported program."""
    L = pkg.load_qsv()
    st = (Step * max(len(steps), 1))(*steps)
    op = (Op * max(len(ops), 1))(*ops)
    pr = (Prim * max(len(prims), 1))(*prims)
    pv = np.ascontiguousarray(pool)
    return L.qsv_program_validate(n_total, n_local, rank, st, len(steps), op, len(ops), pr, len(prims),
                                  pv.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), C.c_size_t(pv.size))


def jit_check(steps, ops, prims, pool, n_total, n_local, rank=0, max_kernels=512):
    """qsv_program_jit_check: host compile + NVRTC sm_100a compile of the pass kernels."""
    L = pkg.load_qsv()
    st = (Step * max(len(steps), 1))(*steps)
    op = (Op * max(len(ops), 1))(*ops)
    pr = (Prim * max(len(prims), 1))(*prims)
    pv = np.ascontiguousarray(pool)
    nk = C.c_int(-1)
    rc = L.qsv_program_jit_check(n_total, n_local, rank, st, len(steps), op, len(ops), pr, len(prims),
                                 pv.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), C.c_size_t(pv.size),
                                 max_kernels, C.byref(nk))
    return rc, nk.value
