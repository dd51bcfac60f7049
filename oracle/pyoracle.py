"""ctypes view of oracle/liboracle.so (CPU restatement, TEST INFRASTRUCTURE ONLY)
and of oracle/_ref/libqsim_ref.so (the reference's own gate.cpp/memtrack.cpp).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        p = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(p):
            raise RuntimeError(f"{p} missing: run `make oracle/liboracle.so`")
        _lib = C.CDLL(p)
    return _lib


def ref_lib():
    """The compiled reference (None when oracle/_ref was not built)."""
    global _ref
    if _ref is None:
        p = os.path.join(_HERE, "_ref", "libqsim_ref.so")
        if not os.path.exists(p):
            return None
        _ref = C.CDLL(p)
    return _ref


def _d(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def threads() -> int:
    return lib().orc_default_threads()


def run_local(circuit, amps: np.ndarray | None = None, nthreads: int | None = None) -> np.ndarray:
    """Reference run_local on the CPU. `circuit` is a package Circuit."""
    n, recs, nr, pool = circuit.export()
    if amps is None:
        amps = np.zeros(1 << n, dtype=np.complex128)
        amps[0] = 1.0
    a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    rc = lib().orc_run_local(n, recs, C.c_int64(nr), _d(pool.view(np.float64)), _d(a.view(np.float64)),
                             nthreads or threads())
    if rc != 0:
        raise RuntimeError(f"orc_run_local failed ({rc})")
    return a


def dense_oracle(circuit, amps: np.ndarray | None = None) -> np.ndarray:
    n, recs, nr, pool = circuit.export()
    if amps is None:
        amps = np.zeros(1 << n, dtype=np.complex128)
        amps[0] = 1.0
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    out = np.empty_like(a)
    rc = lib().orc_dense_oracle(n, recs, C.c_int64(nr), _d(pool.view(np.float64)), _d(a.view(np.float64)),
                                _d(out.view(np.float64)))
    if rc != 0:
        raise RuntimeError(f"orc_dense_oracle failed ({rc})")
    return out


def apply_single(amps: np.ndarray, t: int, u: np.ndarray, mode: str = "grouped", nthreads: int = 1):
    a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    n = int(np.log2(a.size))
    uu = np.ascontiguousarray(u, dtype=np.complex128)
    if mode == "naive":
        rc = lib().orc_apply_single_naive(n, _d(a.view(np.float64)), t, _d(uu.view(np.float64)))
    else:
        rc = lib().orc_apply_single_grouped(n, _d(a.view(np.float64)), t, _d(uu.view(np.float64)), nthreads)
    if rc != 0:
        raise RuntimeError("apply_single failed")
    return a


def apply_controlled(amps: np.ndarray, c: int, t: int, u: np.ndarray, nthreads: int = 1):
    a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    n = int(np.log2(a.size))
    uu = np.ascontiguousarray(u, dtype=np.complex128)
    rc = lib().orc_apply_controlled(n, _d(a.view(np.float64)), c, t, _d(uu.view(np.float64)), nthreads)
    if rc != 0:
        raise RuntimeError("apply_controlled failed")
    return a


def apply_multi(amps: np.ndarray, targets, m: np.ndarray, controls=(), nthreads: int = 1):
    a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    n = int(np.log2(a.size))
    mm = np.ascontiguousarray(m, dtype=np.complex128)
    t = (C.c_int * len(targets))(*targets)
    cc = (C.c_int * max(len(controls), 1))(*controls)
    rc = lib().orc_apply_multi(n, _d(a.view(np.float64)), len(targets), t, len(controls), cc,
                               _d(mm.view(np.float64)), nthreads)
    if rc != 0:
        raise RuntimeError("apply_multi failed")
    return a
