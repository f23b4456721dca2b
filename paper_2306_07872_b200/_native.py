"""ctypes binding of ``libdawn.so`` (the C ABI declared in ``include/dawn.h``).

This module is the only place Python touches the native library.  There is
no CPU fallback: if the library is missing or no CUDA device is visible, the
solvers raise ``RuntimeError`` — the product path never routes through the
oracle.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint, c_uint32, c_uint64, c_void_p
from pathlib import Path

import os

# DAWN_LIB: developer override to load an alternative build (tuning variants)
LIB_PATH = Path(os.environ.get("DAWN_LIB") or Path(__file__).resolve().with_name("libdawn.so"))

DAWN_OK = 0
DAWN_EINVAL = 1
DAWN_ESOURCE = 2
DAWN_ECUDA = 3
DAWN_ENOMEM = 4
DAWN_EUNSUPPORTED = 5

I32, I64, F32, F64 = 0, 1, 2, 3
VTYPE_NAMES = {I32: "int32", I64: "int64", F32: "float32", F64: "float64"}
PREC_AUTO, PREC_FP32, PREC_FP64 = 0, 1, 2
PRECISIONS = {"auto": PREC_AUTO, "exact": PREC_AUTO, "fp32": PREC_FP32, "fp64": PREC_FP64}
GOVM, GSVM = 0, 1
F_PRED = 1
F_NEGCHECK = 2
F_PROFILE = 4
F_ASYNC = 8

# every symbol include/dawn.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "dawn_abi_version",
    "dawn_last_error",
    "dawn_device_count",
    "dawn_choose_vtype",
    "dawn_graph_create",
    "dawn_graph_destroy",
    "dawn_graph_info",
    "dawn_solver_create",
    "dawn_solver_destroy",
    "dawn_solver_tune",
    "dawn_sssp",
    "dawn_sssp_begin",
    "dawn_sssp_advance",
    "dawn_sssp_run",
    "dawn_solver_state",
    "dawn_solver_result",
    "dawn_solver_round_profile",
    "dawn_solver_cta_profile",
    "dawn_solver_worklist_stats",
    "dawn_floyd_warshall",
    "dawn_format_rows",
    "dawn_mssp",
    "dawn_batch_supported",
    "dawn_mssp_batch",
    "dawn_build_csr",
    "dawn_gen_rmat",
    "dawn_gen_grid",
    "dawn_oracle_dijkstra",
    "dawn_oracle_bellman_ford",
)


class Stats(ctypes.Structure):
    """Mirror of ``dawn_stats_t``."""

    _fields_ = [
        ("outer_steps", c_int64),
        ("relaxations", c_int64),
        ("writes", c_int64),
        ("first_discoveries", c_int64),
        ("multi_written", c_int64),
        ("negative_cycle", c_int32),
        ("early_exit", c_int32),
    ]


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def _declare(L: ctypes.CDLL) -> None:
    P64 = POINTER(c_int64)
    PD = POINTER(c_double)
    sig = {
        "dawn_abi_version": (c_int, []),
        "dawn_last_error": (c_char_p, []),
        "dawn_device_count": (c_int, [POINTER(c_int)]),
        "dawn_choose_vtype": (c_int, [c_int64, c_int64, c_void_p, c_int, POINTER(c_int)]),
        "dawn_graph_create": (c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int, c_int, POINTER(c_void_p)]),
        "dawn_graph_destroy": (c_int, [c_void_p]),
        "dawn_graph_info": (c_int, [c_void_p, P64, P64, POINTER(c_int), P64]),
        "dawn_solver_create": (c_int, [c_void_p, c_uint, POINTER(c_void_p)]),
        "dawn_solver_destroy": (c_int, [c_void_p]),
        "dawn_solver_tune": (c_int, [c_void_p, c_char_p, c_double]),
        "dawn_sssp": (c_int, [c_void_p, c_int64, c_int, c_uint, c_void_p, c_void_p, POINTER(Stats), c_void_p]),
        "dawn_sssp_begin": (c_int, [c_void_p, c_int64, c_int, c_uint, c_void_p]),
        "dawn_sssp_advance": (c_int, [c_void_p, c_int, P64, POINTER(c_int), c_void_p]),
        "dawn_sssp_run": (c_int, [c_void_p, c_int, c_void_p]),
        "dawn_solver_state": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
        "dawn_solver_result": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(Stats), c_void_p]),
        "dawn_solver_round_profile": (c_int, [c_void_p, c_void_p, c_int64, P64, c_void_p]),
        "dawn_solver_cta_profile": (c_int, [c_void_p, c_void_p, c_int64, POINTER(c_int), c_void_p]),
        "dawn_solver_worklist_stats": (c_int, [c_void_p, c_void_p, c_void_p]),
        "dawn_floyd_warshall": (c_int, [c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int),
                                        c_void_p]),
        "dawn_format_rows": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int64,
                                     POINTER(c_int64), c_int]),
        "dawn_mssp": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_uint, c_void_p, c_void_p, c_void_p]),
        "dawn_batch_supported": (c_int, [c_void_p, c_int, c_uint, POINTER(c_int)]),
        "dawn_mssp_batch": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_uint, c_void_p, c_int, c_int64,
                                    c_void_p, c_void_p]),
        "dawn_build_csr": (c_int, [c_int, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                   c_void_p, c_void_p]),
        "dawn_gen_rmat": (c_int, [c_int, c_int, c_int64, c_double, c_double, c_double, c_uint64, c_int,
                                  c_int64, c_int64, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p]),
        "dawn_gen_grid": (c_int, [c_int, c_int64, c_int64, c_int, c_int64, c_int64, c_uint64, c_void_p, c_void_p,
                                  c_void_p, c_void_p]),
        "dawn_oracle_dijkstra": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, P64]),
        "dawn_oracle_bellman_ford": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, P64,
                                             POINTER(c_int)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> ctypes.CDLL:
    """Load (once) and return the native library; raise if it is not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise RuntimeError(
                        f"{LIB_PATH.name} is not built (python -m paper_2306_07872_b200.build); "
                        "weighted DAWN has no CPU fallback"
                    )
                L = ctypes.CDLL(str(LIB_PATH))
                _declare(L)
                _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a DAWN status code onto the reference's exception conventions."""
    if rc == DAWN_OK:
        return
    msg = (lib().dawn_last_error() or b"").decode(errors="replace")
    if rc in (DAWN_EINVAL, DAWN_ESOURCE):
        raise ValueError(msg)
    if rc == DAWN_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libdawn error {rc}: {msg}")


def device_count() -> int:
    c = c_int(0)
    rc = lib().dawn_device_count(ctypes.byref(c))
    return c.value if rc == DAWN_OK else 0


def require_gpu() -> None:
    if device_count() < 1:
        raise RuntimeError("weighted DAWN requires a CUDA device (there is no CPU fallback)")
