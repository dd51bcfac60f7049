"""OpenQASM 2.0 subset ingestion / export.

Known answers are the SPEC [OP] examples; the round-trip and
fuzz properties are SPEC:212-215.  The oracle (tests only) checks statevector actions.
"""
import math

import numpy as np
import pytest

import paper_2509_04955_b200 as pkg
from oracle import pyoracle as O

from .helpers import rand_state, random_mnemonic_circuit, random_unitary_circuit


def records(c):
    """(n, [(arity, targets, controls)], pool) with exact matrices."""
    n, recs, nr, pool = c.export()
    out = []
    off = []
    for i in range(nr):
        r = recs[i]
        out.append((r.arity, tuple(r.targets[: r.arity if r.arity else 8]), tuple(r.controls[: r.nctrl])))
        off.append(r.mat_off)
    return n, out, pool


def same_circuit(a, b):
    na, ra, pa = records(a)
    nb, rb, pb = records(b)
    assert na == nb
    assert ra == rb
    # matrices bit-identical (the emitter prints %.17g)
    assert pa.view(np.uint64).tobytes() == pb.view(np.uint64).tobytes()


def test_bell_pair():
    c = pkg.Circuit.from_qasm("OPENQASM 2.0; qreg q[2]; h q[0]; cx q[0],q[1];")
    ref = pkg.Circuit.empty(2).add("h", [0]).add("cx", [0, 1])
    same_circuit(c, ref)


def test_swap_lowers_to_three_cx():
    c = pkg.Circuit.from_qasm("OPENQASM 2.0;\nqreg q[2];\nswap q[0],q[1];\n")
    ref = pkg.Circuit.empty(2).add("cx", [0, 1]).add("cx", [1, 0]).add("cx", [0, 1])
    same_circuit(c, ref)


def test_emit_single_h():
    s = pkg.Circuit.empty(1).add("h", [0]).to_qasm()
    lines = [ln for ln in s.splitlines() if not ln.startswith("//")]
    assert lines == ['OPENQASM 2.0;', 'include "qelib1.inc";', "qreg q[1];", "h q[0];"]


@pytest.mark.parametrize("seed", range(100))
def test_round_trip_random(seed):  # parse(emit(C)) == C for 100 random circuits
    c = random_mnemonic_circuit(2 + seed % 7, 40, seed)
    same_circuit(pkg.Circuit.from_qasm(c.to_qasm()), c)


@pytest.mark.parametrize("spec", ["qft:8", "hea:6:2:4", "qaoa:6:2:1", "random:7:4:2", "uccsd:8:60:3"])
def test_round_trip_generators(spec):  # SPEC:177 (QFT(8)) and the other generator families
    c = pkg.Circuit.generate(spec)
    same_circuit(pkg.Circuit.from_qasm(c.to_qasm()), c)


def test_fused_matrix_export():  # fused gate → identical matrix on reparse
    c = pkg.Circuit.generate("random:6:4:9")
    f = c.fused(pkg.PlanOptions(fuse_k=2, register_blocks=False))
    with pytest.raises(ValueError):
        f.to_qasm()  # inexpressible without matrix export
    r = pkg.Circuit.from_qasm(f.to_qasm(matrix_export=True))
    same_circuit(r, f)
    a = rand_state(6, 1)
    assert np.abs(O.run_local(r, a) - O.run_local(c, a)).max() < 1e-12


def test_unitary_directive_with_controls():
    c = random_unitary_circuit(5, 12, 4, kmax=3, ctrl=True)
    r = pkg.Circuit.from_qasm(c.to_qasm(matrix_export=True))
    same_circuit(r, c)


def test_semantic_identity_small_n():  # parse∘emit action equal within 1e-12, n ≤ 8
    for seed in range(5):
        c = random_mnemonic_circuit(8, 60, 100 + seed)
        r = pkg.Circuit.from_qasm(c.to_qasm())
        a = rand_state(8, seed)
        assert np.abs(O.run_local(r, a) - O.run_local(c, a)).max() <= 1e-12


def test_expressions_and_broadcast():
    c = pkg.Circuit.from_qasm(
        'OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg r[3];\n'
        "rz(pi/2) r[0];\nrx(-pi/4*2) r[1];\nry(2^-1) r[2];\np(sin(pi/6)+cos(0)-1) r[0];\n"
        "h r;  // broadcast\nbarrier r;\ncp(.5e1) r[2], r[0];\n"
    )
    ref = (
        pkg.Circuit.empty(3)
        .add("rz", [0], [math.pi / 2])
        .add("rx", [1], [-math.pi / 4 * 2])
        .add("ry", [2], [0.5])
        .add("p", [0], [math.sin(math.pi / 6) + math.cos(0) - 1])
        .add("h", [0]).add("h", [1]).add("h", [2])
        .add_barrier([0, 1, 2])
        .add("cp", [2, 0], [5.0])
    )
    same_circuit(c, ref)


ERRORS = [
    # (text, line, col, fragment)
    ("OPENQASM 2.0;\nqreg q[2];\nh q[0] @;\n", 3, 8, "unexpected character"),
    ("OPENQASM 2.0;\nqreg q[2];\nu3(1,2,3) q[0];\n", 3, 1, "unknown gate mnemonic"),
    ("OPENQASM 2.0;\nqreg q[2];\ncx q[0];\n", 3, 1, "takes 2 qubit"),
    ("OPENQASM 2.0;\nqreg q[2];\nrz q[0];\n", 3, 1, "parameter"),
    ("OPENQASM 2.0;\nqreg q[2];\nh q[5];\n", 3, 5, "out of range"),
    ("OPENQASM 2.0;\nh q[0];\n", 2, 1, "missing qreg"),
    ("OPENQASM 2.0;\n", 2, 1, "missing qreg"),
    ("OPENQASM 2.0;\nqreg q[2];\ncreg c[2];\n", 3, 1, "not supported"),
    ("OPENQASM 2.0;\nqreg q[2];\nmeasure q[0] -> c[0];\n", 3, 1, "not supported"),
    ("OPENQASM 2.0;\nqreg q[2];\nif (c==1) x q[0];\n", 3, 1, "not supported"),
    ("OPENQASM 2.0;\ninclude \"other.inc\";\n", 2, 9, "not supported"),
    ("OPENQASM 3.0;\n", 1, 10, "only OPENQASM 2.0"),
    ("OPENQASM 2.0;\nqreg q[2];\nqreg r[2];\n", 3, 1, "only one qreg"),
    ("OPENQASM 2.0;\nqreg q[2];\ncx q[1],q[1];\n", 3, 9, "repeated"),
    ("OPENQASM 2.0;\nqreg q[2];\nh p[0];\n", 3, 3, "unknown register"),
    ("OPENQASM 2.0;\nqreg q[2];\nrx(foo) q[0];\n", 3, 4, "unknown identifier"),
    ("OPENQASM 2.0;\nqreg q[2];\nh q[0]\n", 4, 1, "expected ',' or ';'"),
    ("OPENQASM 2.0;\nqreg q[2];\ncx q;\n", 3, 1, "takes 2 qubit"),
    ("OPENQASM 2.0;\nqreg q[2];\ncx q, q[1];\n", 3, 4, "broadcast"),
    ("OPENQASM 2.0;\nqreg q[2];\nrx(1/0) q[0];\n", 3, 5, "division by zero"),
    ("OPENQASM 2.0;\nqreg q[0];\n", 2, 8, ">= 1"),
    ("OPENQASM 2.0;\nqreg q[2];\n// qsv-unitary \"U\" (1, 0) q[0];\n", 3, 20, "needs 8 numbers"),
]


@pytest.mark.parametrize("text,line,col,frag", ERRORS)
def test_located_diagnostics(text, line, col, frag):
    with pytest.raises(pkg.QasmError) as ei:
        pkg.Circuit.from_qasm(text)
    e = ei.value
    assert frag in str(e), str(e)
    assert (e.line, e.column) == (line, col), str(e)
    assert str(e).startswith(f"qasm:{line}:{col}:")


def test_fuzz_never_crashes():  # 10,000 mutated inputs, every failure located
    rng = np.random.default_rng(574)
    seeds = [pkg.Circuit.generate(s).to_qasm().encode() for s in ("qft:5", "hea:4:2:1", "qaoa:4:1:2")]
    seeds.append(random_unitary_circuit(3, 3, 1).to_qasm(matrix_export=True).encode())
    alphabet = np.frombuffer(b"qreg[](),;.-+*/^pi \n\"//barrier swap cx h rz 0123456789e\x00\xff", dtype=np.uint8)
    ok = bad = 0
    for i in range(10_000):
        b = bytearray(seeds[i % len(seeds)])
        for _ in range(int(rng.integers(1, 6))):
            op = rng.integers(0, 4)
            pos = int(rng.integers(0, len(b) + 1))
            if op == 0 and len(b) > 0:
                del b[min(pos, len(b) - 1)]
            elif op == 1:
                b.insert(pos, int(rng.choice(alphabet)))
            elif op == 2 and len(b) > 0:
                b[min(pos, len(b) - 1)] = int(rng.integers(0, 256))
            else:
                cut = int(rng.integers(0, len(b) + 1))
                b = b[:cut]
        try:
            pkg.Circuit.from_qasm(bytes(b))
            ok += 1
        except pkg.QasmError as e:
            assert e.line >= 1 and e.column >= 1, str(e)
            bad += 1
    assert ok + bad == 10_000
    assert bad > 1000 and ok > 100  # the mutations exercise both outcomes


def test_generate_from_file(tmp_path):  # the `qasm:<file>` generator spec (bench / CLI input)
    c = pkg.Circuit.generate("qft:6")
    p = tmp_path / "qft6.qasm"
    p.write_text(c.to_qasm())
    same_circuit(pkg.Circuit.generate(f"qasm:{p}"), c)
    with pytest.raises(ValueError):
        pkg.Circuit.generate(f"qasm:{tmp_path / 'missing.qasm'}")
