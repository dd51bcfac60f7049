import numpy as np
"""The C-ABI libraries load and export every function their headers declare
(no compute calls: runs without a GPU)."""
import ctypes as C
import os
import re

import pytest

import paper_2509_04955_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b((?:qsv|qsim)_\w+)\s*\(", text, flags=re.M)))


@pytest.mark.parametrize("header,loader", [("qsv.h", pkg.load_qsv), ("qsim_c.h", pkg.load_qsim)])
def test_every_declared_symbol_is_exported(header, loader):
    lib = loader()
    names = declared(header)
    assert len(names) > 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_libqsv_is_sm100a_and_has_no_cpu_path():
    # the shared object carries sm_100a SASS for the pass kernel
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pkg.lib_paths()["qsv"]], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_fails_loudly():
    # With no GPU (this container) context creation must fail, not fall back.
    L = pkg.load_qsv()
    n = C.c_int(-1)
    rc = L.qsv_device_count(C.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a GPU is present")
    ctx = C.c_void_p()
    assert L.qsv_ctx_create(0, 0, 1, None, C.byref(ctx)) != 0
    c = pkg.Circuit.generate("qft:4")
    with pytest.raises(Exception):
        pkg.Engine(c)


def test_program_validate_rejects_bad_programs():
    L = pkg.load_qsv()

    class Step(C.Structure):
        _fields_ = [("kind", C.c_int32), ("tile_k", C.c_int32), ("nhigh", C.c_int32), ("high", C.c_int32 * 8),
                    ("op_begin", C.c_int32), ("op_count", C.c_int32), ("has_relabel", C.c_int32),
                ("relabel", C.c_int32 * 16), ("swap_global", C.c_int32),
                    ("swap_local", C.c_int32), ("chunk_log2", C.c_int32), ("nbuf", C.c_int32)]

    class Op(C.Structure):
        _fields_ = [("kind", C.c_int32), ("k", C.c_int32), ("qubits", C.c_int32 * 8), ("ctrl_mask", C.c_uint64),
                    ("mat_off", C.c_int64), ("prim_begin", C.c_int32), ("nprim", C.c_int32),
                ("qmask", C.c_uint64)]

    pool = (C.c_double * 8)(0.0, 0.0, 1.0, 0.0, 1.0, 0.0, 0.0, 0.0)  # X
    op = Op(kind=0, k=1, ctrl_mask=0, mat_off=0)
    op.qubits[0] = 12
    st = Step(kind=0, tile_k=10, nhigh=1, op_begin=0, op_count=1)
    st.high[0] = 12
    assert L.qsv_program_validate(16, 16, 0, C.byref(st), 1, C.byref(op), 1, None, 0, pool, C.c_size_t(4)) == 0
    st.nhigh = 0  # target 12 no longer inside the tile
    assert L.qsv_program_validate(16, 16, 0, C.byref(st), 1, C.byref(op), 1, None, 0, pool, C.c_size_t(4)) == -1
    st.nhigh = 1
    op.mat_off = 3  # matrix outside the pool
    assert L.qsv_program_validate(16, 16, 0, C.byref(st), 1, C.byref(op), 1, None, 0, pool, C.c_size_t(4)) == -1


def test_plan_export_capacity_checked():
    """the second qsim_plan_export call checks the caller's capacities."""
    import ctypes as C
    import paper_2509_04955_b200 as pkg
    from tests import dist_emulator as E
    c = pkg.Circuit.generate("random:12:6:2")
    L = pkg.load_qsim()
    o = pkg.PlanOptions().to_c()
    ns, no, npr, pl = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    assert L.qsim_plan_export(c._h, C.byref(o), 12, C.byref(ns), C.byref(no), C.byref(npr), C.byref(pl),
                              None, None, None, None) == 0
    need = no.value
    assert need >= 2
    ops = (E.Op * need)()
    no.value = need - 1  # too small
    rc = L.qsim_plan_export(c._h, C.byref(o), 12, C.byref(ns), C.byref(no), C.byref(npr), C.byref(pl),
                            None, ops, None, None)
    assert rc != 0 and no.value == need


def test_gather_cap_refused_without_gpu(monkeypatch):
    """a state above the single-host cap is not gathered (checked before any GPU work)."""
    import ctypes as C
    import paper_2509_04955_b200 as pkg
    monkeypatch.setenv("QSV_GATHER_CAP_GIB", "0.000001")
    c = pkg.Circuit.generate("qft:12")
    out = np.zeros(1 << 12, dtype=np.complex128)
    o = pkg.PlanOptions().to_c()
    rc = pkg.load_qsim().qsim_run_distributed(c._h, 1, 8, 2, None, C.byref(o),
                                              out.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), None)
    assert rc != 0 and b"cap" in pkg.load_qsim().qsim_last_error()


def test_background_jit_entry_points_validate_arguments():
    """qsv_program_jit_async / _wait and qsim_engine_jit_wait reject null handles (no device
    needed), and PlanOptions(jit=2) reaches the C struct unchanged."""
    Q, L = pkg.load_qsv(), pkg.load_qsim()
    assert Q.qsv_program_jit_async(None, 8) != 0
    done = C.c_int(-1)
    assert Q.qsv_program_jit_wait(None, 1, C.byref(done), None) != 0
    assert L.qsim_engine_jit_wait(None) != 0
    assert pkg.PlanOptions(jit=2).to_c().jit == 2
    assert pkg.PlanOptions().to_c().jit == 1
