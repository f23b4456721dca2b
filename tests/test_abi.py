"""The C ABI library builds, loads and exports every symbol include/dawn.h declares.
CPU only: no compute call needs a GPU here."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2306_07872_b200 import _native as N
from paper_2306_07872_b200.build import LIB, build

HEADER = Path(__file__).resolve().parent.parent / "include" / "dawn.h"


def header_symbols() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"^(?:int|const char\*)\s+(dawn_\w+)\s*\(", text, flags=re.M))


@pytest.fixture(scope="module")
def lib():
    build()
    return N.lib()


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 15
    assert syms == set(N.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dawn_\w+)", out))
    assert syms <= exported, syms - exported


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_errors(lib):
    assert lib.dawn_abi_version() == 1
    c = ctypes.c_int(-1)
    lib.dawn_device_count(ctypes.byref(c))
    assert c.value >= 0
    rc = lib.dawn_graph_create(0, -1, 0, None, None, None, 0, 0, ctypes.byref(ctypes.c_void_p()))
    assert rc == N.DAWN_EINVAL
    assert b"bad graph" in lib.dawn_last_error()


@pytest.mark.parametrize(
    "vals,prec,expect",
    [
        ([1.0, 2.0, 100.0], N.PREC_AUTO, N.I32),
        ([1.5, 2.0], N.PREC_AUTO, N.F64),
        ([-3.0, 7.0], N.PREC_AUTO, N.I32),
        ([3e9, 1.0], N.PREC_AUTO, N.I64),
        ([1e300, 1.0], N.PREC_AUTO, N.F64),
        ([1.0, 2.0], N.PREC_FP32, N.F32),
        ([1.0, 2.0], N.PREC_FP64, N.F64),
    ],
)
def test_precision_policy(lib, vals, prec, expect):
    a = np.asarray(vals, dtype=np.float64)
    vt = ctypes.c_int(-1)
    assert lib.dawn_choose_vtype(10, a.size, a.ctypes.data, prec, ctypes.byref(vt)) == 0
    assert vt.value == expect


def test_precision_bound_switches_to_int64(lib):
    # n * max|w| must fit int32 for the int32 path (dist after r rounds <= r*max|w|)
    a = np.asarray([1000.0], dtype=np.float64)
    vt = ctypes.c_int(-1)
    lib.dawn_choose_vtype(3_000_000, 1, a.ctypes.data, N.PREC_AUTO, ctypes.byref(vt))
    assert vt.value == N.I64
