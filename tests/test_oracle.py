"""The CPU oracle (oracle/) against the SPEC known answers, the analytic QFT and
the independent explicit-matrix dense oracle (SURVEY §8c chain of trust 1-2)."""
import math

import numpy as np
import pytest

import paper_2509_04955_b200 as pkg
from oracle import pyoracle as O
from tests.helpers import (qft_basis_expected, rand_state, rand_unitary, random_mnemonic_circuit,
                           random_unitary_circuit)

H = np.array([[1, 1], [1, -1]], dtype=complex) / math.sqrt(2)
X = np.array([[0, 1], [1, 0]], dtype=complex)


def test_spec_h_on_zero():
    a = np.array([1, 0], dtype=complex)
    out = O.apply_single(a, 0, H, "naive")
    np.testing.assert_allclose(out, [1 / math.sqrt(2), 1 / math.sqrt(2)], atol=1e-15)


def test_spec_x_on_qubit1():
    a = np.zeros(4, dtype=complex)
    a[0] = 1
    out = O.apply_single(a, 1, X, "grouped")
    assert out[2] == 1 and np.count_nonzero(out) == 1


@pytest.mark.parametrize("t", [0, 1, 2])
def test_spec_random_u_vs_kronecker(t):
    rng = np.random.default_rng(t)
    u = rand_unitary(1, rng)
    a = rand_state(3, t)
    full = np.eye(1)
    for q in reversed(range(3)):
        full = np.kron(full, u if q == t else np.eye(2))
    np.testing.assert_allclose(O.apply_single(a, t, u, "naive"), full @ a, atol=1e-12)


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_grouped_bitwise_equals_naive(threads):
    rng = np.random.default_rng(5)
    a = rand_state(14, 1)
    for t in (0, 5, 13):
        u = rand_unitary(1, rng)
        assert np.array_equal(O.apply_single(a, t, u, "naive"), O.apply_single(a, t, u, "grouped", threads))


def test_cx_fires_and_not():
    a = np.zeros(4, dtype=complex)
    a[1] = 1  # |01>: qubit0 = 1
    out = O.apply_controlled(a, 0, 1, X)
    assert out[3] == 1
    b = np.zeros(4, dtype=complex)
    b[2] = 1  # |10>: control qubit0 = 0
    assert np.array_equal(O.apply_controlled(b, 0, 1, X), b)


@pytest.mark.parametrize("c,t", [(0, 3), (3, 0), (1, 2), (2, 1)])
def test_random_cu_vs_dense(c, t):  # SPEC:83, c > t role swap SPEC:138
    rng = np.random.default_rng(c * 7 + t)
    u = rand_unitary(1, rng)
    a = rand_state(4, c + t)
    circ = pkg.Circuit.empty(4).add_unitary(u, [t], [c])
    np.testing.assert_allclose(O.apply_controlled(a, c, t, u), O.dense_oracle(circ, a), atol=1e-12)
    # control-0 amplitudes are bit-identical before/after
    out = O.apply_controlled(a, c, t, u)
    idx = [i for i in range(16) if not (i >> c) & 1]
    assert np.array_equal(out[idx], a[idx])


def test_apply_multi_known_answers():
    a = np.zeros(4, dtype=complex)
    a[0] = 1
    assert O.apply_multi(a, [0, 1], np.kron(X, X))[3] == 1
    b = rand_state(3, 2)
    assert np.array_equal(O.apply_multi(b, [0, 2], np.eye(4)), b)
    rng = np.random.default_rng(9)
    m = rand_unitary(2, rng)
    circ = pkg.Circuit.empty(3).add_unitary(m, [0, 2])
    np.testing.assert_allclose(O.apply_multi(b, [0, 2], m), O.dense_oracle(circ, b), atol=1e-12)


def test_dense_oracle_examples():
    a = rand_state(3, 4)
    assert np.array_equal(O.dense_oracle(pkg.Circuit.empty(3), a), a)
    c = pkg.Circuit.empty(1).add("h", [0])
    np.testing.assert_allclose(O.dense_oracle(c), [1 / math.sqrt(2)] * 2, atol=1e-15)


@pytest.mark.parametrize("seed", range(40))
def test_run_local_vs_dense_oracle_mnemonics(seed):  # acceptance #1
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 9))
    c = random_mnemonic_circuit(n, int(rng.integers(1, 51)), seed)
    a = rand_state(n, seed)
    assert np.abs(O.run_local(c, a) - O.dense_oracle(c, a)).max() < 1e-10


@pytest.mark.parametrize("seed", range(12))
def test_run_local_vs_dense_oracle_unitaries(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 9))
    c = random_unitary_circuit(n, 20, seed)
    a = rand_state(n, seed)
    assert np.abs(O.run_local(c, a) - O.dense_oracle(c, a)).max() < 1e-10


@pytest.mark.parametrize("n", [4, 10, 16])
def test_qft_of_zero_is_uniform(n):  # SPEC:112, :567 (acceptance #2)
    out = O.run_local(pkg.Circuit.generate(f"qft:{n}"))
    np.testing.assert_allclose(out, np.full(1 << n, 2 ** (-n / 2)), atol=1e-12)


@pytest.mark.parametrize("n,x", [(5, 17), (8, 0xA5), (11, 1234), (14, 0x2A5A)])
def test_qft_basis_state_analytic(n, x):  # the strong form
    a = np.zeros(1 << n, dtype=complex)
    a[x] = 1
    assert np.abs(O.run_local(pkg.Circuit.generate(f"qft:{n}"), a) - qft_basis_expected(n, x)).max() < 1e-12


def test_norm_after_1000_random_gates():
    c = random_mnemonic_circuit(10, 1000, 3)
    out = O.run_local(c, rand_state(10, 3))
    assert abs(np.vdot(out, out).real - 1) < 1e-12


def test_worker_count_bitwise_determinism():  # SPEC:111, acceptance #10
    c = pkg.Circuit.generate("qaoa:16:2:1")
    outs = [O.run_local(c, None, t) for t in (1, 2, 8)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_dense_oracle_scale_guard():
    with pytest.raises(RuntimeError):
        O.dense_oracle(pkg.Circuit.empty(13).add("h", [0]))


def _flat(circ):
    """(targets, controls, matrix) per gate record of an exported circuit."""
    n, recs, nr, pool = circ.export()
    out = []
    for i in range(nr):
        r = recs[i]
        d = 1 << r.arity
        m = pool[r.mat_off:r.mat_off + d * d]
        out.append((tuple(r.targets[:r.arity]), tuple(r.controls[:r.nctrl]), m.tobytes()))
    return n, out


@pytest.mark.parametrize("spec", ["qft:9", "qaoa:8:2:5", "hea:7:3:2", "random:9:6:4", "uccsd:8:300:3"])
def test_generator_restatement_matches_product(spec):
    """oracle/gen.cpp (the reference arm's circuits, built without the product
    libraries) is gate-for-gate and bit-for-bit the product generator."""
    n0, a = _flat(pkg.Circuit.generate(spec))
    n1, b = _flat(O.generate(spec))
    assert n0 == n1 and len(a) == len(b)
    assert a == b


@pytest.mark.parametrize("spec,bits", [("random:14:8:3", 8), ("uccsd:13:400:2", 6), ("qft:12", 5),
                                       ("hea:12:3:1", 10)])
def test_blocked_run_local_bitwise(spec, bits):
    """The cache-blocked schedule (full-size parity checks) is bitwise the pooled run_local."""
    c = O.generate(spec)
    a = rand_state(c.n, 7)
    ref = O.run_local(c, a)
    got = O.run_local(c, a, blocked=True, block_bits=bits)
    assert np.array_equal(ref, got)


def test_inplace_run_local_and_fill_basis():
    c = O.generate("random:12:4:1")
    a = np.empty(1 << 12, dtype=np.complex128)
    O.fill_basis(a, 5)
    assert a[5] == 1 and np.count_nonzero(a) == 1
    ref = O.run_local(c, a)
    out = O.run_local(c, a, inplace=True)
    assert out is a and np.array_equal(a, ref)
