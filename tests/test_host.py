"""Host-side logic on the CPU: generators, the DAGC/SMGP planner's
semantic preservation through the oracle, and the device compiler's
acceptance of every plan (single- and multi-rank)."""
import math

import numpy as np
import pytest

import paper_2509_04955_b200 as pkg
from oracle import pyoracle as O
from tests.helpers import rand_state, random_mnemonic_circuit, random_unitary_circuit


def test_qft_gate_count():  # n(n+1)/2 + floor(n/2) swaps (3 CX each)
    for n in (1, 4, 5, 24, 36):
        _, nrec, _ = pkg.Circuit.generate(f"qft:{n}").info()
        assert nrec == n * (n + 1) // 2 + 3 * (n // 2)
    assert pkg.Circuit.generate("qft:24").info()[1] == 336


def test_hea_gate_counts():  # SPEC:207 and SURVEY §8a a15
    assert pkg.Circuit.generate("hea:4:1:7").info()[1] == 14
    assert pkg.Circuit.generate("hea:33:5:4").info()[1] == 575


def test_generators_deterministic():
    for spec in ("hea:12:3:5", "qaoa:9:2:3", "random:11:6:2", "uccsd:10:200:3"):
        a = pkg.Circuit.generate(spec).export()
        b = pkg.Circuit.generate(spec).export()
        assert np.array_equal(a[3], b[3])


def test_random_circuit_shape():
    n, nrec, _ = pkg.Circuit.generate("random:30:20:2").info()
    assert n == 30 and nrec == 20 * 30 + 10 * 15 + 10 * 14


def test_uccsd_reaches_cx_target():
    c = pkg.Circuit.generate("uccsd:12:500:3")
    n, recs, nr, _ = c.export()
    cx = sum(1 for i in range(nr) if recs[i].arity == 1 and recs[i].nctrl == 1)
    assert cx >= 500


def test_bad_generator_spec():
    with pytest.raises(ValueError):
        pkg.Circuit.generate("nope:3")
    with pytest.raises(ValueError):
        pkg.Circuit.generate("qft:x")


def test_barrier_and_range_errors():
    c = pkg.Circuit.empty(3)
    with pytest.raises(ValueError):
        c.add("h", [3])
    with pytest.raises(ValueError):
        pkg.Circuit.empty(0)
    c.add_barrier([0, 1])


OPTS = [
    pkg.PlanOptions(),
    pkg.PlanOptions(register_blocks=False),
    pkg.PlanOptions(fuse_k=4, register_blocks=False, tile_k=10),
    pkg.PlanOptions(fuse_k=5, register_blocks=False, pass_budget=500),
    pkg.PlanOptions(fusion=False, multi_op_passes=False),
]
SPECS = ["qft:9", "random:10:8:2", "hea:9:3:4", "uccsd:9:200:3", "qaoa:8:2:1"]


@pytest.mark.parametrize("spec", SPECS)
@pytest.mark.parametrize("oi", range(len(OPTS)))
def test_fusion_preserves_semantics(spec, oi):  # SPEC:312, acceptance #4
    c = pkg.Circuit.generate(spec)
    a = rand_state(c.n, 3)
    f = c.fused(OPTS[oi])
    assert np.abs(O.run_local(f, a) - O.run_local(c, a)).max() < 1e-10


@pytest.mark.parametrize("seed", range(10))
def test_fusion_random_unitaries_and_barriers(seed):
    c = random_unitary_circuit(7, 30, seed, kmax=2)
    c.add_barrier([0, 1, 2])
    c2 = random_mnemonic_circuit(7, 30, seed)
    for cc in (c, c2):
        a = rand_state(7, seed)
        assert np.abs(O.run_local(cc.fused(), a) - O.run_local(cc, a)).max() < 1e-10


def test_fusion_never_adds_ops_and_compresses():
    for spec in ("hea:20:5:3", "qaoa:20:2:1", "random:20:10:2", "qft:20"):
        st = pkg.Circuit.generate(spec).plan()
        assert st["ops_fused"] <= st["gates_in"]
        assert st["ops_final"] <= st["ops_fused"]
        assert st["passes"] < st["gates_in"]


@pytest.mark.parametrize("spec", ["random:30:20:2", "qft:24", "hea:33:5:4", "uccsd:28:20000:3", "qft:36"])
def test_plans_accepted_by_device_compiler(spec):
    st = pkg.Circuit.generate(spec).plan()
    assert st["passes"] >= 1 and st["swaps"] == 0


@pytest.mark.parametrize("spec", ["random:20:10:2", "qft:20", "hea:18:3:4", "uccsd:16:300:3"])
@pytest.mark.parametrize("m", [1, 2, 3])
def test_multi_rank_plans_accepted(spec, m):  # partition into 2^m ranks
    c = pkg.Circuit.generate(spec)
    for rank in range(1 << m):
        st = c.plan(n_local=c.n - m, rank=rank)
        assert st["n_local"] == c.n - m


def test_qft_collapses_phase_chains():
    st = pkg.Circuit.generate("qft:30").plan()
    # one H + one phase product per qubit (plus the swap layer)
    assert st["ops_fused"] <= 30 + 30 + 45
