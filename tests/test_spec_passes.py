"""SPEC-level host passes: build_dag, gate_cost and the DAGC
rules / contract, SMGP planning, partitioning
(SPEC:359-377).  CPU only; semantics checked through the oracle."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_2509_04955_b200 as pkg
from oracle import pyoracle as O
from tests.helpers import rand_state, random_mnemonic_circuit


class FusionStats(C.Structure):
    _fields_ = [("gates_before", C.c_int64), ("gates_after", C.c_int64), ("merges_same_qubit", C.c_int64),
                ("merges_cu", C.c_int64), ("merges_kronecker", C.c_int64), ("passes", C.c_int64),
                ("compression_ratio", C.c_double), ("cost_before", C.c_double), ("cost_after", C.c_double)]


def L():
    lib = pkg.load_qsim()
    lib.qsim_dag_edges.restype = C.c_int64
    return lib


def edges(c):
    pairs = (C.c_int32 * 4096)()
    n = L().qsim_dag_edges(c._h, pairs, C.c_int64(2048))
    assert n >= 0
    return sorted((pairs[2 * i], pairs[2 * i + 1]) for i in range(n))


def contract(c, cap=2):
    h = C.c_void_p()
    st = FusionStats()
    rc = L().qsim_contract(c._h, cap, C.byref(h), C.byref(st))
    assert rc == 0
    return pkg.Circuit(h.value), st


def mat(c, i=0):
    n, recs, nr, pool = c.export()
    r = recs[i]
    d = 1 << r.arity
    return pool[r.mat_off:r.mat_off + d * d].reshape(d, d), r


def test_dag_examples():
    assert edges(pkg.Circuit.empty(2).add("h", [0]).add("h", [1])) == []
    c = pkg.Circuit.empty(2).add("h", [0]).add("cx", [0, 1]).add("h", [1])
    assert edges(c) == [(0, 1), (1, 2)]
    b = pkg.Circuit.empty(3).add("h", [0]).add_barrier([0, 1, 2]).add("h", [2])
    assert edges(b) == [(0, 1), (1, 2)]


def test_dag_independent_gates_commute():
    c = pkg.Circuit.empty(4).add("rx", [0], [0.3]).add("ry", [2], [1.1])
    d = pkg.Circuit.empty(4).add("ry", [2], [1.1]).add("rx", [0], [0.3])
    a = rand_state(4, 1)
    assert np.abs(O.dense_oracle(c, a) - O.dense_oracle(d, a)).max() < 1e-12


@pytest.mark.parametrize("n", [10, 20])
def test_gate_cost_anchors(n):  # SPEC:267-268, acceptance #5
    c = pkg.Circuit.empty(n).add("h", [0]).add_unitary(np.eye(4), [0, 1]).add("cx", [0, 1])
    v = C.c_double()
    L().qsim_gate_cost(c._h, C.c_int64(0), n, C.byref(v))
    assert v.value == 10 * 2 ** (n - 1)
    L().qsim_gate_cost(c._h, C.c_int64(1), n, C.byref(v))
    assert v.value == 36 * 2 ** (n - 2)
    L().qsim_gate_cost(c._h, C.c_int64(2), n, C.byref(v))
    assert v.value == 5 * 2 ** (n - 1)  # controlled = half (Eq. 4)


def test_fuse_same_qubit_examples():
    f, st = contract(pkg.Circuit.empty(1).add("h", [0]).add("h", [0]))
    m, _ = mat(f)
    np.testing.assert_allclose(m, np.eye(2), atol=1e-15)
    assert st.compression_ratio == 0.5
    f, _ = contract(pkg.Circuit.empty(1).add("x", [0]).add("z", [0]))
    np.testing.assert_allclose(mat(f)[0], [[0, 1], [-1, 0]], atol=0)
    f, _ = contract(pkg.Circuit.empty(1).add("rz", [0], [0.3]).add("rz", [0], [0.5]))
    rz = np.diag([np.exp(-0.4j), np.exp(0.4j)])
    np.testing.assert_allclose(mat(f)[0], rz, atol=1e-12)


def test_fuse_kronecker_examples():
    f, st = contract(pkg.Circuit.empty(2).add("x", [0]).add("x", [1]))
    m, r = mat(f)
    np.testing.assert_allclose(m, np.fliplr(np.eye(4)), atol=0)
    assert [r.targets[0], r.targets[1]] == [0, 1] and st.merges_kronecker == 1
    c = pkg.Circuit.empty(3).add("ry", [0], [0.7]).add("rx", [2], [1.9])
    f, _ = contract(c)
    a = rand_state(3, 2)
    assert np.abs(O.run_local(f, a) - O.run_local(c, a)).max() < 1e-12


def test_fuse_cu_examples():
    f, st = contract(pkg.Circuit.empty(2).add("cx", [0, 1]).add("cx", [0, 1]))
    m, r = mat(f)
    np.testing.assert_allclose(m, np.eye(2), atol=0)
    assert r.nctrl == 1 and st.merges_cu == 1
    f, _ = contract(pkg.Circuit.empty(2).add("cp", [0, 1], [0.2]).add("cp", [0, 1], [0.9]))
    np.testing.assert_allclose(mat(f)[0], np.diag([1, np.exp(1.1j)]), atol=1e-12)


def test_barrier_is_never_crossed():
    c = pkg.Circuit.empty(1).add("h", [0]).add_barrier([0]).add("h", [0])
    f, st = contract(c)
    assert st.gates_after == 2


@pytest.mark.parametrize("seed", range(15))
def test_contract_preserves_semantics_and_cost_decreases(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 9))
    c = random_mnemonic_circuit(n, 40, seed)
    for cap in (2, 3):
        f, st = contract(c, cap)
        a = rand_state(n, seed)
        assert np.abs(O.run_local(f, a) - O.run_local(c, a)).max() < 1e-10
        assert st.cost_after <= st.cost_before
        assert st.gates_after <= st.gates_before
        assert st.compression_ratio == pytest.approx((st.gates_before - st.gates_after) / st.gates_before)


def test_compression_floors():  # SPEC:308-309, acceptance #4 (HEA compresses more than QAOA)
    # Floors are DERIVED from the reconstructed generators as the SPEC prescribes
    # (measured: HEA(20,5) 0.578 vs the paper's 63.07%; ring-QAOA(20,2) 0.178 vs
    # 52.13% — the paper's QAOA instances are unspecified).
    _, hea = contract(pkg.Circuit.generate("hea:20:5:3"))
    _, qaoa = contract(pkg.Circuit.generate("qaoa:20:2:1"))
    assert hea.compression_ratio >= 0.40
    assert qaoa.compression_ratio >= 0.15
    assert hea.compression_ratio > qaoa.compression_ratio


def test_stagger_schedule_latin():  # SPEC:463-465, Table 3
    t = (C.c_int32 * 16)()
    assert L().qsim_stagger_schedule(4, 4, t) == 0
    table = np.array(list(t)).reshape(4, 4)
    assert list(table[1]) == [1, 2, 3, 0]
    for tau in range(4):
        assert len(set(table[:, tau])) == 4
    for g in range(4):
        assert sorted(table[g]) == [0, 1, 2, 3]
    t2 = (C.c_int32 * 8)()
    assert L().qsim_stagger_schedule(2, 4, t2) == 0


def groups_of(c, S, l=-1):
    n, nr, _ = c.info()
    g = (C.c_int32 * max(nr, 1))()
    ng = L().qsim_plan_groups(c._h, S, l, g)
    return ng, list(g)[:nr]


def test_plan_groups_examples():
    ng, g = groups_of(pkg.Circuit.empty(6).add("h", [0]).add("h", [1]).add("h", [2]).add("h", [3]), 4)
    assert ng == 1 and g == [0, 0, 0, 0]
    ng, g = groups_of(pkg.Circuit.empty(4).add("h", [0]).add("cx", [0, 1]), 4)
    assert ng == 0
    ng, g = groups_of(pkg.Circuit.empty(6).add("h", [5]).add("h", [0]), 4)
    assert g[0] == -1


def test_classify_and_peer_rank():
    c = pkg.Circuit.empty(7).add("h", [3]).add("h", [6]).add("cx", [5, 2]).add("cx", [5, 6])
    out = C.c_int()
    kinds = []
    for i in range(4):
        assert L().qsim_classify_gate(c._h, C.c_int64(i), 2, C.byref(out)) == 0
        kinds.append(out.value)
    assert kinds == [0, 1, 2, 3]
    for r, t, l, want in ((0, 5, 5, 1), (2, 6, 5, 0)):
        assert L().qsim_peer_rank(r, t, l, C.byref(out)) == 0 and out.value == want
    for r in range(8):
        L().qsim_peer_rank(r, 6, 4, C.byref(out))
        p = out.value
        L().qsim_peer_rank(p, 6, 4, C.byref(out))
        assert out.value == r
    assert L().qsim_peer_rank(0, 3, 5, C.byref(out)) == -1
