"""Generates tests/golden/reference_fixtures.json from the REFERENCE's own code.

Runs in the build container only (needs /root/reference): oracle/build_ref.sh
compiles /root/reference/proj/src/gate.cpp + memtrack.cpp into oracle/_ref/,
and this script records, through that library,
  * the matrix, targets and controls of every QASM mnemonic (ref gate.cpp:116-200),
  * the unitarity verdict of GateMatrix on a set of near-unitary matrices
    (ref gate.cpp:13-38, tolerance 1e-10),
  * the rejection of bad mnemonics/arity (ref gate.cpp:172-200),
  * peak_bytes after scripted memtrack sessions (ref memtrack.cpp:11-80).
The committed JSON pins the rebuild's API-compatible host code and the oracle's
gate inputs on machines where /root/reference does not exist (the GPU box).
"""
import ctypes as C
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402

MNEMONICS = [
    ("h", [], [0]), ("x", [], [1]), ("y", [], [2]), ("z", [], [0]), ("s", [], [3]), ("sdg", [], [0]),
    ("t", [], [1]), ("tdg", [], [2]), ("rx", [0.7], [0]), ("ry", [1.3], [1]), ("rz", [2.9], [2]),
    ("rx", [-4.1], [3]), ("ry", [math.pi], [0]), ("rz", [1e-3], [1]), ("u1", [0.3], [0]), ("p", [5.5], [2]),
    ("cx", [], [0, 1]), ("cx", [], [3, 1]), ("cz", [], [1, 2]), ("cp", [0.25], [2, 0]),
    ("cu1", [1.75], [0, 3]), ("cp", [math.pi / 8], [4, 5]),
]
BAD = [("foo", [], [0]), ("h", [0.1], [0]), ("rx", [], [0]), ("cx", [], [0]), ("cx", [], [0, 0]),
       ("swap", [], [0, 1]), ("barrier", [], [0])]
MEMTRACK_SCRIPTS = [
    [[0, 2], [1, 0], [3, 100], [3, 50], [4, 120], [3, 10], [2, 1], [3, 7], [1, 1], [3, 999]],
    [[0, 1], [1, 0], [3, 5], [4, 500], [3, 3], [5, 0], [3, 4]],
    [[0, 3], [1, 2], [3, 64], [6, 0], [3, 1000], [1, 5], [3, 7]],
    [[1, 0], [3, 64], [0, 1], [1, 0], [3, 8], [4, 8], [3, 2]],
]


def main():
    ref = pyoracle.ref_lib()
    if ref is None:
        raise SystemExit("oracle/_ref/libqsim_ref.so missing: run oracle/build_ref.sh")
    out = {"source": "reference proj/src/gate.cpp + memtrack.cpp compiled by oracle/build_ref.sh",
           "gates": [], "bad": [], "unitarity": [], "memtrack": []}
    for name, params, qubits in MNEMONICS:
        ar, nt, nc = C.c_int(), C.c_int(), C.c_int()
        tg, ct = (C.c_int * 8)(), (C.c_int * 8)()
        mat = (C.c_double * 512)()
        err = C.create_string_buffer(256)
        rc = ref.ref_gate(name.encode(), (C.c_double * 4)(*params), len(params), (C.c_int * 4)(*qubits), len(qubits),
                          C.byref(ar), tg, C.byref(nt), ct, C.byref(nc), mat, err)
        assert rc == 0, err.value
        d = 1 << ar.value
        out["gates"].append({
            "name": name, "params": params, "qubits": qubits, "arity": ar.value,
            "targets": [tg[i] for i in range(nt.value)], "controls": [ct[i] for i in range(nc.value)],
            # repr() keeps every bit of each double
            "matrix": [[float.hex(mat[2 * i]), float.hex(mat[2 * i + 1])] for i in range(d * d)],
        })
    for name, params, qubits in BAD:
        ar, nt, nc = C.c_int(), C.c_int(), C.c_int()
        tg, ct = (C.c_int * 8)(), (C.c_int * 8)()
        mat = (C.c_double * 512)()
        err = C.create_string_buffer(256)
        rc = ref.ref_gate(name.encode(), (C.c_double * 4)(*params), len(params), (C.c_int * 4)(*qubits), len(qubits),
                          C.byref(ar), tg, C.byref(nt), ct, C.byref(nc), mat, err)
        out["bad"].append({"name": name, "params": params, "qubits": qubits, "rejected": rc != 0})
    rng = np.random.default_rng(7)
    for k in (1, 2, 3):
        d = 1 << k
        q, _ = np.linalg.qr(rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d)))
        for eps in (0.0, 1e-12, 4e-11, 2e-10, 1e-8, 1e-3):
            m = q.copy()
            m[0, 0] += eps
            flat = np.ascontiguousarray(m).reshape(-1).view(np.float64)
            acc = ref.ref_matrix_accepts(k, flat.ctypes.data_as(C.POINTER(C.c_double)))
            out["unitarity"].append({"k": k, "matrix": [float.hex(float(x)) for x in flat], "accepted": bool(acc)})
    ref.ref_memtrack_script.argtypes = [C.POINTER(C.c_longlong), C.c_int, C.c_int, C.POINTER(C.c_ulonglong)]
    for sc in MEMTRACK_SCRIPTS:
        flat = [v for pair in sc for v in pair]
        nranks = 4
        peaks = (C.c_ulonglong * (2 * nranks))()
        ref.ref_memtrack_script((C.c_longlong * len(flat))(*flat), len(sc), nranks, peaks)
        out["memtrack"].append({"script": sc, "nranks": nranks, "peaks": list(peaks)})
    with open(os.path.join(HERE, "reference_fixtures.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out["gates"]), "gates,", len(out["unitarity"]), "unitarity cases,",
          len(out["memtrack"]), "memtrack scripts")


if __name__ == "__main__":
    main()
