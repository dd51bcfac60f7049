"""ctypes view of oracle/liboracle.so (CPU restatement, TEST INFRASTRUCTURE ONLY)
and of oracle/_ref/libqsim_ref.so (the reference's own gate.cpp/memtrack.cpp).
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None
_ref = None
_native = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        p = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(p):
            raise RuntimeError(f"{p} missing: run `make oracle/liboracle.so`")
        _lib = C.CDLL(p)
    return _lib


def native_lib() -> C.CDLL:
    """liboracle built for THIS host (-O3 -march=native -fcx-limited-range)
    into a host-local cache, for the CPU timing legs; the shipped oracle/liboracle.so is
    portable (x86-64-v3) because it is built in one container and run on another host.
    Falls back to the portable library when no compiler is available."""
    global _native
    if _native is not None:
        return _native
    srcs = [os.path.join(_HERE, f) for f in ("oracle.cpp", "gen.cpp", "oracle.h")]
    h = hashlib.sha1()
    for f in srcs:
        with open(f, "rb") as fh:
            h.update(fh.read())
    out_dir = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"qsv_oracle_native_{h.hexdigest()[:12]}")
    out = os.path.join(out_dir, "liboracle_native.so")
    if not os.path.exists(out):
        os.makedirs(out_dir, exist_ok=True)
        tmp = f"{out}.{os.getpid()}"
        cmd = [os.environ.get("CXX", "g++"), "-std=c++20", "-O3", "-march=native", "-fcx-limited-range", "-fPIC",
               "-shared", srcs[0], srcs[1], "-o", tmp, "-lpthread"]
        try:
            subprocess.run(cmd, check=True, capture_output=True, timeout=300)
            os.replace(tmp, out)
        except Exception:
            _native = lib()
            return _native
    _native = C.CDLL(out)
    return _native


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


class orc_gate(C.Structure):
    _fields_ = [("arity", C.c_int32), ("nctrl", C.c_int32), ("targets", C.c_int32 * 8),
                ("controls", C.c_int32 * 8), ("mat_off", C.c_int64)]


MNEMONICS = ("h", "rx", "ry", "rz", "cx", "cp")  # ORC_* codes of oracle.h


def _restated_matrix(name: str, theta: float) -> np.ndarray:
    """Gate matrices as gate.cpp:116-164 writes them (fallback when oracle/_ref is absent)."""
    import math
    if name == "h":
        r = 1.0 / math.sqrt(2.0)
        return np.array([r, r, r, -r], dtype=np.complex128)
    if name == "rx":
        c, s = math.cos(theta / 2), math.sin(theta / 2)
        return np.array([c, -1j * s, -1j * s, c], dtype=np.complex128)
    if name == "ry":
        c, s = math.cos(theta / 2), math.sin(theta / 2)
        return np.array([c, -s, s, c], dtype=np.complex128)
    if name == "rz":
        return np.array([complex(math.cos(-theta / 2), math.sin(-theta / 2)), 0, 0,
                         complex(math.cos(theta / 2), math.sin(theta / 2))], dtype=np.complex128)
    if name == "cx":
        return np.array([0, 1, 1, 0], dtype=np.complex128)
    return np.array([1, 0, 0, complex(math.cos(theta), math.sin(theta))], dtype=np.complex128)


class OracleCircuit:
    """A circuit in the oracle's flat form, built without the product libraries."""

    def __init__(self, n: int, recs, nr: int, pool: np.ndarray, source: str = ""):
        self.n, self.recs, self.nr, self.pool, self.source = n, recs, nr, pool, source

    def export(self):
        return self.n, self.recs, self.nr, self.pool

    def info(self):
        return self.n, self.nr, self.pool.size

    def slice(self, begin: int, end: int) -> "OracleCircuit":
        end = min(end, self.nr)
        recs = (orc_gate * max(end - begin, 1))()
        C.memmove(recs, C.addressof(self.recs) + begin * C.sizeof(orc_gate), (end - begin) * C.sizeof(orc_gate))
        return OracleCircuit(self.n, recs, end - begin, self.pool, self.source)


def generate(spec: str, matrices: str = "auto") -> OracleCircuit:
    """The workload circuit of `spec` (qft|qaoa|hea|random|uccsd) from the restated generators
    (oracle/gen.cpp).  Gate matrices come from the reference's own gates::from_mnemonic
    (oracle/_ref) when it was built, else from the restated table; both are bit-identical
    (tests/test_oracle.py)."""
    L = lib()
    L.orc_generate.restype = C.c_int64
    n = C.c_int()
    cnt = L.orc_generate(spec.encode(), C.byref(n), None, None, None, None, C.c_int64(0))
    if cnt < 0:
        raise ValueError(f"bad generator spec {spec!r}")
    codes = np.zeros(cnt, np.int32)
    q0 = np.zeros(cnt, np.int32)
    q1 = np.zeros(cnt, np.int32)
    params = np.zeros(cnt, np.float64)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    L.orc_generate(spec.encode(), C.byref(n), ip(codes), ip(q0), ip(q1), _d(params), C.c_int64(cnt))
    ref = ref_lib() if matrices in ("auto", "reference") else None
    if matrices == "reference" and ref is None:
        raise RuntimeError("oracle/_ref not built")
    recs = (orc_gate * max(int(cnt), 1))()
    mats: dict = {}
    chunks = []
    off = 0
    for i in range(cnt):
        code, a, b, th = int(codes[i]), int(q0[i]), int(q1[i]), float(params[i])
        name = MNEMONICS[code]
        key = (code, th)
        if key not in mats:
            if ref is not None:
                m = _ref_matrix(ref, name, th, [a] if b < 0 else [a, b])
            else:
                m = _restated_matrix(name, th)
            mats[key] = off
            chunks.append(m)
            off += m.size
        r = recs[i]
        r.arity = 1
        r.mat_off = mats[key]
        if b < 0:
            r.nctrl = 0
            r.targets[0] = a
        else:
            r.nctrl = 1
            r.controls[0] = a
            r.targets[0] = b
    pool = np.concatenate(chunks) if chunks else np.zeros(1, np.complex128)
    return OracleCircuit(n.value, recs, int(cnt), pool, spec)


def _ref_matrix(ref, name: str, theta: float, qubits) -> np.ndarray:
    arity, nt, nc = C.c_int(), C.c_int(), C.c_int()
    tg, ct = (C.c_int * 8)(), (C.c_int * 8)()
    mat = np.zeros(8, np.float64)
    err = C.create_string_buffer(256)
    ps = (C.c_double * 1)(theta)
    qs = (C.c_int * len(qubits))(*qubits)
    npar = 0 if name in ("h", "cx") else 1
    rc = ref.ref_gate(name.encode(), ps, npar, qs, len(qubits), C.byref(arity), tg, C.byref(nt), ct, C.byref(nc),
                      _d(mat), err)
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return mat.view(np.complex128).copy()


def run_local(circuit, amps: np.ndarray | None = None, nthreads: int | None = None, inplace: bool = False,
              blocked: bool = False, block_bits: int = 16, library=None) -> np.ndarray:
    """Reference run_local on the CPU.  `circuit` is a package Circuit or an
    OracleCircuit.  inplace=True updates `amps` (complex128, C-contiguous) without a copy;
    blocked=True uses the bitwise-equal cache-blocked schedule (orc_run_local_blocked)."""
    n, recs, nr, pool = circuit.export()
    if amps is None:
        a = np.zeros(1 << n, dtype=np.complex128)
        a[0] = 1.0
    elif inplace:
        if amps.dtype != np.complex128 or not amps.flags.c_contiguous:
            raise ValueError("inplace run_local needs a C-contiguous complex128 array")
        a = amps
    else:
        a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    L = library or lib()
    if blocked:
        rc = L.orc_run_local_blocked(n, recs, C.c_int64(nr), _d(pool.view(np.float64)), _d(a.view(np.float64)),
                                     nthreads or threads(), block_bits)
    else:
        rc = L.orc_run_local(n, recs, C.c_int64(nr), _d(pool.view(np.float64)), _d(a.view(np.float64)),
                             nthreads or threads())
    if rc != 0:
        raise RuntimeError(f"orc_run_local failed ({rc})")
    return a


def fill_basis(amps: np.ndarray, index: int = 0, nthreads: int | None = None, library=None) -> np.ndarray:
    """|index> into `amps` (complex128, C-contiguous), zero-filled by the worker pool."""
    if amps.dtype != np.complex128 or not amps.flags.c_contiguous:
        raise ValueError("fill_basis needs a C-contiguous complex128 array")
    n = int(amps.size).bit_length() - 1
    if (1 << n) != amps.size:
        raise ValueError("fill_basis needs 2^n amplitudes")
    rc = (library or lib()).orc_fill_basis(n, _d(amps.view(np.float64)), C.c_uint64(index), nthreads or threads())
    if rc != 0:
        raise RuntimeError(f"orc_fill_basis failed ({rc})")
    return amps


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
