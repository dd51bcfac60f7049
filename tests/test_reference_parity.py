"""Pins the API-compatible host code against the reference's own compiled
gate.cpp / memtrack.cpp, via fixtures committed by tests/golden/make_golden.py
(and live against oracle/_ref when it is present)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2509_04955_b200 as pkg
from oracle import pyoracle

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.json")))


def _gate_record(name, params, qubits):
    c = pkg.Circuit.empty(8).add(name, qubits, params)
    n, recs, nr, pool = c.export()
    r = recs[0]
    d = 1 << r.arity
    return r, pool[r.mat_off:r.mat_off + d * d]


@pytest.mark.parametrize("g", FIX["gates"], ids=lambda g: f"{g['name']}{g['qubits']}")
def test_gate_matrices_bit_identical_to_reference(g):  # ref gate.cpp:116-200
    r, mat = _gate_record(g["name"], g["params"], g["qubits"])
    assert r.arity == g["arity"]
    assert [r.targets[i] for i in range(r.arity)] == g["targets"]
    assert [r.controls[i] for i in range(r.nctrl)] == g["controls"]
    want = np.array([complex(float.fromhex(a), float.fromhex(b)) for a, b in g["matrix"]])
    # bit-identical (== treats -0.0 and +0.0 as equal, as the arithmetic does)
    assert np.array_equal(mat, want)


@pytest.mark.parametrize("b", FIX["bad"], ids=lambda b: b["name"])
def test_bad_mnemonics_rejected_like_reference(b):  # ref gate.cpp:172-200
    assert b["rejected"]
    with pytest.raises(ValueError):
        pkg.Circuit.empty(8).add(b["name"], b["qubits"], b["params"])


@pytest.mark.parametrize("i", range(len(FIX["unitarity"])))
def test_unitarity_check_matches_reference(i):  # ref gate.cpp:13-38 (1e-10 per entry)
    u = FIX["unitarity"][i]
    flat = np.array([float.fromhex(x) for x in u["matrix"]]).view(np.complex128)
    d = 1 << u["k"]
    m = flat.reshape(d, d)
    c = pkg.Circuit.empty(4)
    if u["accepted"]:
        c.add_unitary(m, list(range(u["k"])))
    else:
        with pytest.raises(ValueError):
            c.add_unitary(m, list(range(u["k"])))


@pytest.mark.parametrize("i", range(len(FIX["memtrack"])))
def test_memtrack_matches_reference(i):  # ref memtrack.cpp:11-80
    s = FIX["memtrack"][i]
    flat = [v for pair in s["script"] for v in pair]
    L = pkg.load_qsim()
    peaks = (C.c_ulonglong * (2 * s["nranks"]))()
    L.qsim_memtrack_script((C.c_longlong * len(flat))(*flat), len(s["script"]), s["nranks"], peaks)
    assert list(peaks) == s["peaks"]
    L.qsim_memtrack_script((C.c_longlong * 2)(6, 0), 1, 0, peaks)  # disable again


def test_live_reference_agrees_with_fixture():
    ref = pyoracle.ref_lib()
    if ref is None:
        pytest.skip("oracle/_ref not built here (no /root/reference)")
    g = FIX["gates"][8]
    ar, nt, nc = C.c_int(), C.c_int(), C.c_int()
    tg, ct = (C.c_int * 8)(), (C.c_int * 8)()
    mat = (C.c_double * 512)()
    err = C.create_string_buffer(256)
    assert ref.ref_gate(g["name"].encode(), (C.c_double * 4)(*g["params"]), len(g["params"]),
                        (C.c_int * 4)(*g["qubits"]), len(g["qubits"]), C.byref(ar), tg, C.byref(nt), ct,
                        C.byref(nc), mat, err) == 0
    assert [float.hex(mat[i]) for i in range(8)] == [x for pair in g["matrix"] for x in pair]
