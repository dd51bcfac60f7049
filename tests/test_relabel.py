"""Pass relabelling (tile-qubit permutation at pass ends, planner.cpp relabel_tile):
the executed single-rank program, including every relabel step and the final
restore, is replayed by the numpy emulator and compared with the oracle."""
import numpy as np
import pytest

import paper_2509_04955_b200 as pkg
from oracle import pyoracle as O
from tests import dist_emulator as E
from tests.helpers import rand_state

CASES = ["random:12:8:2", "uccsd:11:300:3", "hea:12:4:4", "qft:11", "qaoa:10:2:1", "random:10:12:7"]


def _plans(spec, **kw):
    c = pkg.Circuit.generate(spec)
    o = dict(tile_k=7, min_low=3)
    o.update(kw)
    return c, pkg.PlanOptions(relabel=2, **o), pkg.PlanOptions(relabel=0, **o)


@pytest.mark.parametrize("spec", CASES)
def test_relabel_plan_matches_oracle(spec):
    c, on, _ = _plans(spec)
    steps, ops, prims, pool = E.export_plan(c, on, c.n)
    a = rand_state(c.n, 11)
    psi = E.run_program(a.copy(), steps, ops, prims, pool, 0, c.n, None)
    ref = O.run_local(c, a)
    assert np.abs(psi - ref).max() < 1e-10


def test_relabel_used_and_saves_passes():
    used = 0
    for spec in CASES:
        c, on, off = _plans(spec)
        steps, *_ = E.export_plan(c, on, c.n)
        used += sum(s.has_relabel for s in steps)
        auto = c.plan(pkg.PlanOptions(relabel=1, tile_k=7, min_low=3))["passes"]
        try:
            on6 = c.plan(pkg.PlanOptions(relabel=2, tile_k=7, min_low=6))["passes"]
        except pkg.QsvError:
            on6 = None  # blocks do not fit the longer low run: auto keeps the plain plan
        assert auto in (on6, c.plan(off)["passes"])  # auto: the cheaper of the two by the time model
    assert used > 0


def test_relabel_rejects_non_permutation():
    c, on, _ = _plans("random:12:8:2")
    steps, ops, prims, pool = E.export_plan(c, on, c.n)
    i = next(i for i, s in enumerate(steps) if s.has_relabel)
    steps[i].relabel[1] = steps[i].relabel[0]
    rc = E.validate(steps, ops, prims, pool, c.n, c.n, 0)
    assert rc != 0


@pytest.mark.parametrize("spec", CASES)
@pytest.mark.parametrize("kw", [dict(), dict(tile_k=7, min_low=3), dict(tile_k=8, min_low=4, pass_budget=200.0)])
def test_default_plans_match_oracle(spec, kw):
    """The auto planner (list schedule x relabel, picked by plan_time_model) executed
    step by step by the emulator equals the oracle."""
    c = pkg.Circuit.generate(spec)
    steps, ops, prims, pool = E.export_plan(c, pkg.PlanOptions(**kw), c.n)
    a = rand_state(c.n, 5)
    psi = E.run_program(a.copy(), steps, ops, prims, pool, 0, c.n, None)
    assert np.abs(psi - O.run_local(c, a)).max() < 1e-10


def test_list_schedule_never_worse():
    for spec in ("random:14:10:2", "hea:13:4:4", "qaoa:12:2:1"):
        c = pkg.Circuit.generate(spec)
        on = c.plan(pkg.PlanOptions(tile_k=8))["passes"]
        off = c.plan(pkg.PlanOptions(tile_k=8, list_schedule=False, relabel=0))["passes"]
        assert on <= off


def _swap_heavy(n, seed):
    """Random circuit with explicit SWAP gates (QASM `swap` -> three CX)."""
    rng = np.random.default_rng(seed)
    lines = ["OPENQASM 2.0;", f"qreg q[{n}];"]
    for _ in range(60):
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        k = rng.integers(0, 3)
        if k == 0:
            lines.append(f"swap q[{a}],q[{b}];")
        elif k == 1:
            lines.append(f"rx({rng.uniform(0, 6.28)}) q[{a}];")
        else:
            lines.append(f"cx q[{a}],q[{b}];")
    return pkg.Circuit.from_qasm("\n".join(lines))


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("kw", [dict(logical_swaps=2), dict(tile_k=7, min_low=3, logical_swaps=2),
                                dict(relabel=0, list_schedule=False, logical_swaps=2), dict(tile_k=7, min_low=3)])
def test_logical_swaps_match_oracle(seed, kw):
    """SWAP gates planned as relabellings (logical_swaps) give the oracle's amplitudes."""
    c = _swap_heavy(11, seed)
    steps, ops, prims, pool = E.export_plan(c, pkg.PlanOptions(**kw), c.n)
    a = rand_state(c.n, seed)
    psi = E.run_program(a.copy(), steps, ops, prims, pool, 0, c.n, None)
    assert np.abs(psi - O.run_local(c, a)).max() < 1e-10
    # the fused op list (with swaps re-expanded) is equivalent too
    f = c.fused(pkg.PlanOptions(**kw))
    assert np.abs(O.run_local(f, a) - O.run_local(c, a)).max() < 1e-10
