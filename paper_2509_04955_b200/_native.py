"""ctypes bindings of include/qsv.h and include/qsim_c.h.

Mirrors the reference objects (SPEC = /root/reference/SPEC.md):
``Circuit`` ~ Circuit/Gate/from_mnemonic (ref gate.hpp:33-92),
generators, ``Engine`` ~ run_local with the state
resident in HBM, ``run_local_host`` ~ run_local on host amplitudes.
Errors: QSV_E_ARG -> ValueError (the reference's std::invalid_argument),
anything else -> QsvError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBDIR = os.path.join(_HERE, "lib")

QSV_OK = 0
QSV_E_ARG = -1


class QsvError(RuntimeError):
    pass


def lib_paths() -> dict:
    return {
        "qsv": os.path.join(_LIBDIR, "libqsv.so"),
        "qsim": os.path.join(_LIBDIR, "libqsim.so"),
    }


class qsim_gate_rec(C.Structure):
    _fields_ = [
        ("arity", C.c_int32),
        ("nctrl", C.c_int32),
        ("targets", C.c_int32 * 8),
        ("controls", C.c_int32 * 8),
        ("mat_off", C.c_int64),
    ]


class qsim_plan_opts(C.Structure):
    _fields_ = [
        ("tile_k", C.c_int32),
        ("min_low", C.c_int32),
        ("fuse_k", C.c_int32),
        ("fusion", C.c_int32),
        ("multi_op_passes", C.c_int32),
        ("chunk_log2", C.c_int32),
        ("nbuf", C.c_int32),
        ("register_blocks", C.c_int32),
        ("pass_budget", C.c_double),
        ("rblock_k", C.c_int32),
        ("jit", C.c_int32),
        ("relabel", C.c_int32),
        ("max_sweeps", C.c_double),
        ("list_schedule", C.c_int32),
        ("jit_max_kernels", C.c_int32),
        ("logical_swaps", C.c_int32),
    ]


class qsv_trace_rec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("step", C.c_int32), ("chunk", C.c_int32), ("stream", C.c_int32),
                ("start_ms", C.c_double), ("end_ms", C.c_double)]


class qsim_plan_stats(C.Structure):
    _fields_ = [
        ("gates_in", C.c_int64),
        ("ops_lowered", C.c_int64),
        ("ops_fused", C.c_int64),
        ("ops_final", C.c_int64),
        ("passes", C.c_int64),
        ("swaps", C.c_int64),
        ("cost_units", C.c_double),
        ("max_dense_k", C.c_int32),
        ("n", C.c_int32),
        ("n_local", C.c_int32),
        ("nsteps", C.c_int32),
    ]

    def as_dict(self) -> dict:
        return {f[0]: getattr(self, f[0]) for f in self._fields_}


_qsv = None
_qsim = None


def load_qsv() -> C.CDLL:
    """libqsv.so (the CUDA C-ABI). Raises if the extension was not built."""
    global _qsv
    if _qsv is None:
        p = lib_paths()["qsv"]
        if not os.path.exists(p):
            raise QsvError(f"{p} missing: build the CUDA extension (python -c 'import __graft_entry__ as g; g.build()')")
        _qsv = C.CDLL(p, mode=C.RTLD_GLOBAL)
        _qsv.qsv_last_error.restype = C.c_char_p
        _qsv.qsv_ctx_stream.restype = C.c_void_p
    return _qsv


def load_qsim() -> C.CDLL:
    """libqsim.so (host library + facade); loads libqsv.so first."""
    global _qsim
    if _qsim is None:
        load_qsv()
        p = lib_paths()["qsim"]
        if not os.path.exists(p):
            raise QsvError(f"{p} missing: build the host library")
        L = C.CDLL(p)
        L.qsim_last_error.restype = C.c_char_p
        for f in ("qsim_engine_stream", "qsim_engine_qsv_state", "qsim_engine_qsv_program", "qsim_engine_qsv_ctx"):
            getattr(L, f).restype = C.c_void_p
            getattr(L, f).argtypes = [C.c_void_p]
        L.qsim_circuit_free.argtypes = [C.c_void_p]
        L.qsim_engine_free.argtypes = [C.c_void_p]
        _qsim = L
    return _qsim


class QasmError(ValueError):
    """A QASM parse error with its 1-based location (qsim::QasmError)."""

    def __init__(self, message: str, line: int, column: int):
        super().__init__(message)
        self.line = line
        self.column = column


def _check(rc: int, what: str, lib=None) -> None:
    if rc == QSV_OK:
        return
    lib = lib or load_qsim()
    msg = (lib.qsim_last_error() if hasattr(lib, "qsim_last_error") else lib.qsv_last_error()) or b""
    text = f"{what}: {msg.decode(errors='replace')} (code {rc})"
    if rc == QSV_E_ARG:
        raise ValueError(text)
    raise QsvError(text)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class PlanOptions:
    tile_k: int = 11
    min_low: int = 5
    fuse_k: int = 2
    fusion: bool = True
    multi_op_passes: bool = True
    chunk_log2: int = 26
    nbuf: int = 2
    pass_budget: float = 120.0
    register_blocks: bool = True
    rblock_k: int = 4
    jit: int = True  # True/1 specialised kernels, 2 compiled in the background (interpreted runs until loaded), 0 off
    relabel: int = 1  # 0 off, 1 auto (kept when it saves passes), 2 always
    max_sweeps: float = 8.0
    list_schedule: bool = True
    jit_max_kernels: int = 8192
    logical_swaps: int = 0  # 0 off, 1 when the time model prefers it, 2 always

    @classmethod
    def default(cls) -> "PlanOptions":
        o = qsim_plan_opts()
        load_qsim().qsim_default_opts(C.byref(o))
        return cls(o.tile_k, o.min_low, o.fuse_k, bool(o.fusion), bool(o.multi_op_passes),
                   o.chunk_log2, o.nbuf, o.pass_budget, bool(o.register_blocks), o.rblock_k, o.jit if o.jit == 2 else bool(o.jit),
                   int(o.relabel), o.max_sweeps, bool(o.list_schedule), o.jit_max_kernels,
                   int(o.logical_swaps))

    def to_c(self) -> qsim_plan_opts:
        return qsim_plan_opts(self.tile_k, self.min_low, self.fuse_k, int(self.fusion),
                              int(self.multi_op_passes), self.chunk_log2, self.nbuf,
                              int(self.register_blocks), float(self.pass_budget), int(self.rblock_k),
                              int(self.jit), int(self.relabel), float(self.max_sweeps),
                              int(self.list_schedule), int(self.jit_max_kernels), int(self.logical_swaps))


class Circuit:
    """Owns a qsim::Circuit (C++)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    # -- construction -----------------------------------------------------
    @classmethod
    def generate(cls, spec: str) -> "Circuit":
        h = C.c_void_p()
        _check(load_qsim().qsim_circuit_generate(spec.encode(), C.byref(h)), f"generate({spec})")
        return cls(h.value)

    @classmethod
    def empty(cls, n: int) -> "Circuit":
        h = C.c_void_p()
        _check(load_qsim().qsim_circuit_new(n, C.byref(h)), "qsim_circuit_new")
        return cls(h.value)

    @classmethod
    def from_qasm(cls, text: str | bytes) -> "Circuit":
        """parse_qasm; raises QasmError(line, column) on bad input."""
        b = text.encode() if isinstance(text, str) else bytes(text)
        h = C.c_void_p()
        line = C.c_int()
        col = C.c_int()
        L = load_qsim()
        rc = L.qsim_circuit_parse_qasm(C.c_char_p(b), C.c_int64(len(b)), C.byref(h), C.byref(line), C.byref(col))
        if rc != QSV_OK:
            msg = (L.qsim_last_error() or b"").decode(errors="replace")
            if rc == QSV_E_ARG:
                raise QasmError(msg, line.value, col.value)
            _check(rc, "parse_qasm")
        return cls(h.value)

    def to_qasm(self, matrix_export: bool = False) -> str:
        """emit_qasm."""
        L = load_qsim()
        need = C.c_int64()
        _check(L.qsim_circuit_emit_qasm(self._h, int(matrix_export), None, C.c_int64(0), C.byref(need)), "emit_qasm")
        buf = C.create_string_buffer(need.value + 1)
        _check(L.qsim_circuit_emit_qasm(self._h, int(matrix_export), buf, C.c_int64(need.value + 1), C.byref(need)),
               "emit_qasm")
        return buf.value.decode()

    def add(self, mnemonic: str, qubits, params=()) -> "Circuit":
        q = (C.c_int * len(qubits))(*qubits)
        p = (C.c_double * max(len(params), 1))(*params)
        _check(load_qsim().qsim_circuit_add(self._h, mnemonic.encode(), p, len(params), q, len(qubits)),
               f"add({mnemonic})")
        return self

    def add_unitary(self, matrix: np.ndarray, targets, controls=(), label: str = "U") -> "Circuit":
        m = np.ascontiguousarray(np.asarray(matrix, dtype=np.complex128)).view(np.float64)
        k = len(targets)
        t = (C.c_int * k)(*targets)
        cc = (C.c_int * max(len(controls), 1))(*controls)
        _check(load_qsim().qsim_circuit_add_unitary(self._h, k, t, len(controls), cc, _dptr(m), label.encode()),
               "add_unitary")
        return self

    def add_barrier(self, qubits) -> "Circuit":
        q = (C.c_int * max(len(qubits), 1))(*qubits)
        _check(load_qsim().qsim_circuit_add_barrier(self._h, len(qubits), q), "add_barrier")
        return self

    # -- inspection -------------------------------------------------------
    def info(self):
        n = C.c_int()
        nr = C.c_int64()
        pl = C.c_int64()
        _check(load_qsim().qsim_circuit_info(self._h, C.byref(n), C.byref(nr), C.byref(pl)), "info")
        return n.value, nr.value, pl.value

    @property
    def n(self) -> int:
        return self.info()[0]

    def export(self):
        """(n, records[np.void], pool[complex128]) — the flat form the oracle consumes."""
        n, nr, pl = self.info()
        recs = (qsim_gate_rec * max(nr, 1))()
        pool = np.zeros(max(pl, 1), dtype=np.complex128)
        _check(load_qsim().qsim_circuit_export(self._h, recs, _dptr(pool.view(np.float64))), "export")
        return n, recs, nr, pool

    def inverse(self) -> "Circuit":
        """C^dagger: the gates in reverse order with adjoint matrices (barriers dropped);
        C followed by C^dagger maps every state to itself (mirror-circuit checks)."""
        n, recs, nr, pool = self.export()
        out = Circuit.empty(n)
        for i in reversed(range(nr)):
            r = recs[i]
            if r.arity == 0:
                continue
            d = 1 << r.arity
            m = pool[r.mat_off:r.mat_off + d * d].reshape(d, d)
            out.add_unitary(m.conj().T, list(r.targets[:r.arity]), list(r.controls[:r.nctrl]), "INV")
        return out

    def concat(self, other: "Circuit") -> "Circuit":
        """This circuit followed by `other` (same qubit count)."""
        n, recs, nr, pool = self.export()
        n2, recs2, nr2, pool2 = other.export()
        if n != n2:
            raise ValueError("concat: qubit counts differ")
        out = Circuit.empty(n)
        for rr, k, pl in ((recs, nr, pool), (recs2, nr2, pool2)):
            for i in range(k):
                r = rr[i]
                if r.arity == 0:
                    continue
                d = 1 << r.arity
                out.add_unitary(pl[r.mat_off:r.mat_off + d * d].reshape(d, d), list(r.targets[:r.arity]),
                                list(r.controls[:r.nctrl]), "G")
        return out

    def slice(self, begin: int, end: int) -> "Circuit":
        h = C.c_void_p()
        _check(load_qsim().qsim_circuit_slice(self._h, C.c_int64(begin), C.c_int64(end), C.byref(h)), "slice")
        return Circuit(h.value)

    def fused(self, opts: PlanOptions | None = None) -> "Circuit":
        h = C.c_void_p()
        o = (opts or PlanOptions()).to_c()
        _check(load_qsim().qsim_circuit_fused(self._h, C.byref(o), C.byref(h)), "fused")
        return Circuit(h.value)

    def plan(self, opts: PlanOptions | None = None, n_local: int = -1, rank: int = 0) -> dict:
        s = qsim_plan_stats()
        o = (opts or PlanOptions()).to_c()
        _check(load_qsim().qsim_circuit_plan(self._h, C.byref(o), n_local, rank, C.byref(s)), "plan")
        return s.as_dict()

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _qsim is not None:
            _qsim.qsim_circuit_free(self._h)
            self._h = C.c_void_p()


class Engine:
    """A planned circuit on one GPU (one rank) with its HBM-resident state shard."""

    def __init__(self, circuit: Circuit, opts: PlanOptions | None = None, device: int = 0,
                 rank: int = 0, nranks: int = 1, comm_id: bytes | None = None):
        L = load_qsim()
        h = C.c_void_p()
        o = (opts or PlanOptions()).to_c()
        cid = C.create_string_buffer(comm_id, 128) if comm_id else None
        _check(L.qsim_engine_create(circuit._h, C.byref(o), device, rank, nranks, cid, C.byref(h)),
               "qsim_engine_create")
        self._h = h
        self.n = circuit.n
        st = qsim_plan_stats()
        _check(L.qsim_engine_stats(self._h, C.byref(st)), "stats")
        self.stats = st.as_dict()
        self.n_local = st.n_local

    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        rc = load_qsv().qsv_comm_unique_id(buf)
        _check(rc, "qsv_comm_unique_id", load_qsv())
        return buf.raw

    @property
    def stream(self) -> int:
        return load_qsim().qsim_engine_stream(self._h)

    def set_basis(self, index: int = 0):
        _check(load_qsim().qsim_engine_set_basis(self._h, C.c_uint64(index)), "set_basis")

    def upload(self, amps: np.ndarray, offset: int = 0):
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        _check(load_qsim().qsim_engine_upload(self._h, _dptr(a.view(np.float64)), C.c_uint64(offset),
                                              C.c_uint64(a.size)), "upload")

    def download(self, offset: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        count = (1 << self.n_local) - offset if count is None else count
        a = np.empty(count, dtype=np.complex128) if out is None else out
        _check(load_qsim().qsim_engine_download(self._h, _dptr(a.view(np.float64)), C.c_uint64(offset),
                                                C.c_uint64(count)), "download")
        return a

    def run(self):
        _check(load_qsim().qsim_engine_run(self._h), "run")

    def sync(self):
        _check(load_qsim().qsim_engine_sync(self._h), "sync")

    def time(self, iters: int, basis: int = -1) -> float:
        """Device ms for `iters` runs (each preceded by a reset to |basis> when basis >= 0)."""
        ms = C.c_float()
        _check(load_qsim().qsim_engine_time(self._h, iters, C.c_int64(basis), C.byref(ms)), "time")
        return ms.value

    def norm_sq(self) -> float:
        v = C.c_double()
        _check(load_qsim().qsim_engine_norm_sq(self._h, C.byref(v)), "norm_sq")
        return v.value

    def max_abs_diff(self, ref: np.ndarray, offset: int = 0) -> float:
        a = np.ascontiguousarray(ref, dtype=np.complex128)
        v = C.c_double()
        _check(load_qsim().qsim_engine_max_abs_diff(self._h, _dptr(a.view(np.float64)), C.c_uint64(offset),
                                                    C.c_uint64(a.size), C.byref(v)), "max_abs_diff")
        return v.value

    def check_qft(self, x: int) -> float:
        v = C.c_double()
        _check(load_qsim().qsim_engine_check_qft(self._h, C.c_uint64(x), C.byref(v)), "check_qft")
        return v.value

    def digest(self) -> int:
        v = C.c_uint64()
        _check(load_qsim().qsim_engine_digest(self._h, C.byref(v)), "digest")
        return v.value

    def steps(self) -> list[dict]:
        L = load_qsim()
        out = []
        for i in range(L.qsim_engine_nsteps(self._h)):
            kind, nops = C.c_int(), C.c_int()
            hbm, fl, nvl = C.c_double(), C.c_double(), C.c_double()
            _check(L.qsim_engine_step_info(self._h, i, C.byref(kind), C.byref(nops), C.byref(hbm),
                                           C.byref(fl), C.byref(nvl)), "step_info")
            out.append({"kind": "pass" if kind.value == 0 else "swap", "nops": nops.value,
                        "hbm_bytes": hbm.value, "flops": fl.value, "nvl_bytes": nvl.value})
        return out

    def jit_info(self) -> dict:
        k, s = C.c_int(), C.c_double()
        _check(load_qsim().qsim_engine_jit_info(self._h, C.byref(k), C.byref(s)), "jit_info")
        return {"kernels": k.value, "seconds": s.value}

    def jit_wait(self):
        """Waits for a background compile (PlanOptions(jit=2)) and switches to its kernels."""
        _check(load_qsim().qsim_engine_jit_wait(self._h), "jit_wait")

    def profile(self) -> list[float]:
        n = load_qsim().qsim_engine_nsteps(self._h)
        ms = (C.c_float * max(n, 1))()
        _check(load_qsim().qsim_engine_profile(self._h, ms), "profile")
        return [ms[i] for i in range(n)]

    TRACE_KINDS = {0: "pass", 1: "swap", 2: "sendrecv", 3: "copyback", 4: "barrier"}

    def trace_enable(self, on: bool = True):
        """PipelineTrace: bracket every launch / swap chunk with CUDA events."""
        _check(load_qsv().qsv_trace_enable(C.c_void_p(load_qsim().qsim_engine_qsv_ctx(self._h)), int(on)),
               "qsv_trace_enable", load_qsv())

    def trace(self) -> list[dict]:
        """The trace since trace_enable: [{kind, step, chunk, stream, start_ms, end_ms}]."""
        L = load_qsv()
        ctx = C.c_void_p(load_qsim().qsim_engine_qsv_ctx(self._h))
        n = C.c_int()
        _check(L.qsv_trace_read(ctx, None, 0, C.byref(n)), "qsv_trace_read", L)
        recs = (qsv_trace_rec * max(n.value, 1))()
        _check(L.qsv_trace_read(ctx, recs, n.value, C.byref(n)), "qsv_trace_read", L)
        return [{"kind": self.TRACE_KINDS.get(r.kind, str(r.kind)), "step": r.step, "chunk": r.chunk,
                 "stream": ("compute", "comm", "copy")[r.stream], "start_ms": r.start_ms, "end_ms": r.end_ms}
                for r in recs[:n.value]]

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            load_qsim().qsim_engine_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_local_host(circuit: Circuit, amps: np.ndarray, opts: PlanOptions | None = None) -> np.ndarray:
    """Reference-facing run_local on host amplitudes (in place on a copy)."""
    a = np.ascontiguousarray(amps, dtype=np.complex128).copy()
    o = (opts or PlanOptions()).to_c()
    _check(load_qsim().qsim_run_local_host(circuit._h, C.byref(o), _dptr(a.view(np.float64))), "run_local_host")
    return a
