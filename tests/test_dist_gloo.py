"""Multi-rank host logic on CPU (world_size 2, gloo): the planner's partition +
swap insertion, rank-bit controls/diagonals, and the chunked qubit-swap
protocol of swap.cu, executed by a numpy emulator and compared with the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2509_04955_b200 as pkg
from oracle import pyoracle as O
from tests.helpers import rand_state

CASES = [
    ("qft:10", {}),
    ("random:11:8:2", {}),
    ("hea:10:3:4", {"chunk_log2": 3, "nbuf": 1}),
    ("uccsd:10:200:3", {"chunk_log2": 2, "nbuf": 3}),
    ("random:12:6:5", {"register_blocks": False}),
    ("qaoa:9:2:1", {"fusion": False, "multi_op_passes": False}),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, kw, q):
    import torch
    from tests import dist_emulator as E

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = pkg.Circuit.generate(spec)
        n = c.n
        m = world.bit_length() - 1
        l = n - m
        opts = pkg.PlanOptions(tile_k=min(8, l), **kw)
        steps, ops, prims, pool = E.export_plan(c, opts, l)
        a = rand_state(n, 7)
        psi = a[rank << l:(rank + 1) << l].copy()

        def exchange(psi, g, v, chunk_log2, nbuf):
            peer = rank ^ (1 << (g - l))
            chunks = E.swap_indices(l, rank, g, v, chunk_log2)
            for ch in chunks:  # grouped send/recv per chunk, like ncclSend/ncclRecv
                send = torch.from_numpy(np.ascontiguousarray(psi[ch]).view(np.float64).copy())
                recv = torch.empty_like(send)
                reqs = [dist.isend(send, peer), dist.irecv(recv, peer)]
                for r in reqs:
                    r.wait()
                psi[ch] = recv.numpy().view(np.complex128)

        E.run_program(psi, steps, ops, prims, pool, rank, l, exchange)
        out = [torch.zeros(2 << l, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(psi.view(np.float64).copy()))
        if rank == 0:
            full = np.concatenate([o.numpy().view(np.complex128) for o in out])
            ref = O.run_local(c, a)
            nswaps = sum(1 for s in steps if s.kind == 1)
            q.put((float(np.abs(full - ref).max()), nswaps))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec,kw", CASES, ids=[c[0] for c in CASES])
def test_two_rank_plan_matches_oracle(spec, kw):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, spec, kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    err, nswaps = q.get(timeout=5)
    assert err < 1e-10
    assert nswaps >= 1  # the global qubit was touched, so the plan exchanged data


def test_two_rank_logical_swaps(tmp_path):
    """A circuit full of SWAP gates, planned with SWAPs as relabellings (logical_swaps=2),
    across two ranks: global qubits move through relabelling as well as qubit swaps."""
    rng = np.random.default_rng(9)
    lines = ["OPENQASM 2.0;", "qreg q[11];"]
    for _ in range(50):
        a, b = (int(x) for x in rng.choice(11, 2, replace=False))
        k = rng.integers(0, 3)
        lines.append(f"swap q[{a}],q[{b}];" if k == 0 else
                     (f"ry({rng.uniform(0, 6.28)}) q[{a}];" if k == 1 else f"cx q[{a}],q[{b}];"))
    path = tmp_path / "swaps.qasm"
    path.write_text("\n".join(lines))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, f"qasm:{path}", {"logical_swaps": 2}, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    err, nswaps = q.get(timeout=5)
    assert err < 1e-10


@pytest.mark.parametrize("spec", ["random:12:6:2", "hea:11:3:4", "uccsd:10:200:3"])
def test_program_order_plan_same_on_every_p(spec):
    """with list scheduling off, the multi-rank planner applies the ops in program
    order (swaps only in between), so every P sees the same op sequence as one GPU."""
    from tests import dist_emulator as E
    c = pkg.Circuit.generate(spec).fused(pkg.PlanOptions())
    o = pkg.PlanOptions(fusion=False, list_schedule=False, relabel=0, register_blocks=False)

    def seq(n_local):
        steps, ops, prims, pool = E.export_plan(c, o, n_local)
        out = []
        for st in steps:
            if st.kind != 0:
                continue
            for op in ops[st.op_begin:st.op_begin + st.op_count]:
                d = {0: 1 << (2 * op.k), 1: 1 << op.k}.get(op.kind, 0)
                out.append((op.kind, op.k, pool[op.mat_off:op.mat_off + d].tobytes()))
        return out

    one = seq(c.n)
    for m in (1, 2):
        got = seq(c.n - m)
        assert got[:len(one)] == one
        for kind, k, data in got[len(one):]:  # the final layout restore: exact permutations
            v = np.frombuffer(data, dtype=np.complex128)
            assert kind == 0 and set(np.unique(v)) <= {0, 1}


def _insert_zero(x, p):
    lo = x & ((1 << p) - 1)
    return ((x ^ lo) << 1) | lo


def _multi_swap_emulated(shards, l, gs, vs):
    """numpy restatement of csrc/swap.cu run_multi_swap + p2p_swap_region_kernel index math:
    for each step s, rank r pairs with the rank whose g bits are (its g bits) ^ s; the pair
    swaps r's block (v bits = partner's g bits) with the partner's block (v bits = r's g bits),
    r doing the first half of the pairs when r < partner."""
    k = len(gs)
    R = len(shards)
    pos = sorted(vs)
    pairs = 1 << (l - k)
    half = pairs // 2
    gmask = sum(1 << (g - l) for g in gs)
    todo = []
    for r in range(R):
        mybits = sum(((r >> (g - l)) & 1) << i for i, g in enumerate(gs))
        for sx in range(1, 1 << k):
            y = mybits ^ sx
            q = r & ~gmask
            for i, g in enumerate(gs):
                q |= ((y >> i) & 1) << (g - l)
            mine_v = sum(((y >> i) & 1) << vs[i] for i in range(k))
            theirs_v = sum(((mybits >> i) & 1) << vs[i] for i in range(k))
            begin = 0 if r < q else half
            todo.append((r, q, begin, mine_v, theirs_v))
    for r, q, begin, mine_v, theirs_v in todo:
        for i in range(begin, begin + half):
            x = i
            for p in pos:
                x = _insert_zero(x, p)
            a, b = x | mine_v, x | theirs_v
            shards[r][a], shards[q][b] = shards[q][b].copy(), shards[r][a].copy()
    return shards


def _pair_swap_emulated(shards, l, g, v):
    R = len(shards)
    for r in range(R):
        q = r ^ (1 << (g - l))
        if r > q:
            continue
        # rank r (bit 0) gives its bit-v = 1 half, receives the peer's bit-v = 0 half
        for i in range(1 << (l - 1)):
            x = _insert_zero(i, v)
            shards[r][x | (1 << v)], shards[q][x] = shards[q][x].copy(), shards[r][x | (1 << v)].copy()
    return shards


@pytest.mark.parametrize("k", [2, 3])
def test_multi_swap_index_math(k):
    """The merged k-qubit remap (k = 3 needs 8 GPUs, more than the test pool offers) moves every
    amplitude where k pairwise swaps would: checked on the host with the kernel's index math."""
    l = 6
    R = 1 << k
    rng = np.random.default_rng(k)
    base = [rng.normal(size=1 << l) + 1j * rng.normal(size=1 << l) for _ in range(R)]
    gs = [l + i for i in range(k)]
    vs = [5, 1, 3][:k]
    merged = _multi_swap_emulated([b.copy() for b in base], l, gs, vs)
    seq = [b.copy() for b in base]
    for g, v in zip(gs, vs):
        seq = _pair_swap_emulated(seq, l, g, v)
    for a, b in zip(merged, seq):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("x", [0, 0b1010011, 0b1111111, 0b0100100])
def test_basis_start_swap_relabel_index_math(x):
    """csrc/qsv_capi.cu enqueue_steps: leading qubit swaps on a basis state |x> become x with
    bits g and v exchanged (the single 1 moves; no transfer).  Checked on the host against the
    pairwise swap's data movement (the kernel's index math) for a run of swaps on 4 ranks."""
    l, R = 5, 4
    shards = [np.zeros(1 << l, dtype=np.complex128) for _ in range(R)]
    shards[x >> l][x & ((1 << l) - 1)] = 1.0
    seq = [(5, 2), (6, 0), (5, 4)]  # (global g, local v) in program order
    moved = shards
    for g, v in seq:
        moved = _pair_swap_emulated(moved, l, g, v)
    y = x
    for g, v in seq:
        if ((y >> g) & 1) != ((y >> v) & 1):
            y ^= (1 << g) | (1 << v)
    want = [np.zeros(1 << l, dtype=np.complex128) for _ in range(R)]
    want[y >> l][y & ((1 << l) - 1)] = 1.0
    for a, b in zip(moved, want):
        assert np.array_equal(a, b)
