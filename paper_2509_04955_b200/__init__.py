"""B200-native full-amplitude state-vector simulator (arXiv 2509.04955 hot path).

The package is a thin Python view of two in-tree native libraries:

* ``lib/libqsv.so``  — sm_100a CUDA kernels behind the C-ABI ``include/qsv.h``
* ``lib/libqsim.so`` — the C++ host library (the reference's ``proj/include``
  qsim API, the DAGC/SMGP planner, the device engine) with the C facade
  ``include/qsim_c.h``

There is no Python or CPU compute path: every amplitude update runs in the
CUDA library, and importing the bindings fails loudly when it is missing.
"""
from ._native import (  # noqa: F401
    QSV_OK,
    Circuit,
    Engine,
    PlanOptions,
    QasmError,
    QsvError,
    lib_paths,
    load_qsim,
    load_qsv,
    run_local_host,
)

__all__ = [
    "Circuit",
    "Engine",
    "PlanOptions",
    "QasmError",
    "QsvError",
    "lib_paths",
    "load_qsim",
    "load_qsv",
    "run_local_host",
]
