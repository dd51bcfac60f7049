"""The NVRTC path on CPU: every distinct specialised pass kernel a plan would
JIT (jit.cu gen_ops / kernel_source) must compile for sm_100a.  NVRTC needs no
device, so generator bugs surface here rather than as a silent interpreter
fallback on the GPU box."""
import os

import pytest

import paper_2509_04955_b200 as pkg
from tests import dist_emulator as E


def _nvrtc_present():
    import ctypes.util
    return any(os.path.exists(os.path.join(d, "libnvrtc.so")) for d in ("/usr/local/cuda/lib64",)) or \
        ctypes.util.find_library("nvrtc") is not None


CASES = [
    ("random:16:8:2", dict()),
    ("random:16:8:2", dict(relabel=2)),
    ("random:14:6:3", dict(relabel=2, tile_k=8, min_low=4)),
    ("uccsd:14:400:3", dict(relabel=2)),
    ("qft:14", dict()),
    ("qaoa:13:2:1", dict()),
    ("hea:15:3:4", dict(rblock_k=3)),
    ("random:14:6:2", dict(register_blocks=False, fuse_k=4, tile_k=10)),
    ("random:14:6:2", dict(register_blocks=False, fuse_k=5, pass_budget=500)),
    ("random:16:8:2", dict(tile_k=12, relabel=2)),
    ("qft:16", dict(tile_k=12)),
]


@pytest.mark.skipif(not _nvrtc_present(), reason="libnvrtc not in this image")
def test_split_blocks_compile(monkeypatch):
    monkeypatch.setenv("QSV_JIT_SPLIT", "1")  # opt-in variant: two threads per register group
    c = pkg.Circuit.generate("random:16:8:2")
    steps, ops, prims, pool = E.export_plan(c, pkg.PlanOptions(), c.n)
    rc, nk = E.jit_check(steps, ops, prims, pool, c.n, c.n)
    assert rc == 0, pkg.load_qsv().qsv_last_error()


@pytest.mark.skipif(not _nvrtc_present(), reason="libnvrtc not in this image")
@pytest.mark.parametrize("spec,kw", CASES)
def test_jit_kernels_compile(spec, kw):
    # the cubin cache is keyed by the full generated source, so a cached hit is a
    # compile of identical text; any generator change recompiles through NVRTC
    c = pkg.Circuit.generate(spec)
    steps, ops, prims, pool = E.export_plan(c, pkg.PlanOptions(**kw), c.n)
    rc, nk = E.jit_check(steps, ops, prims, pool, c.n, c.n)
    assert rc == 0, pkg.load_qsv().qsv_last_error()
    assert nk >= 1


@pytest.mark.skipif(not _nvrtc_present(), reason="libnvrtc not in this image")
def test_class_mode_kernels_compile(monkeypatch):
    """Structure-class kernels (QSV_JIT_CLASS_MIN): runtime masks, rolled primitive switch."""
    monkeypatch.setenv("QSV_JIT_CLASS_MIN", "0")
    c = pkg.Circuit.generate("uccsd:14:400:3")
    steps, ops, prims, pool = E.export_plan(c, pkg.PlanOptions(relabel=2), c.n)
    rc, nk = E.jit_check(steps, ops, prims, pool, c.n, c.n)
    assert rc == 0, pkg.load_qsv().qsv_last_error()
    assert 1 <= nk < len([s for s in steps if s.kind == 0])
