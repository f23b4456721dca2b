"""ctypes wrapper of the CPU oracle (``oracle/dawn_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's CPU-baseline / ``--impl reference`` legs — never by the product
package (``paper_2306_07872_b200``), which has no CPU fallback.

* :func:`gs_sssp`      — the reference's Gauss-Seidel order in float64,
                         reference counters (solver.py:212-399).
* :func:`jacobi_sssp`  — snapshot-Jacobi restatement in the device value
                         type; the exact distances/counters the GPU reports.
* :func:`gs_multi`     — k independent reference-order solves on T threads
                         (the timed CPU baseline).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
SRC = HERE / "dawn_oracle.c"

VTYPES = {"int32": 0, "int64": 1, "float32": 2, "float64": 3, "i32": 0, "i64": 1, "f32": 2, "f64": 3}


class OStats(ctypes.Structure):
    _fields_ = [
        ("outer_steps", c_int64),
        ("relaxations", c_int64),
        ("writes", c_int64),
        ("first_discoveries", c_int64),
        ("multi_written", c_int64),
        ("negative_cycle", c_int32),
        ("early_exit", c_int32),
    ]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "-B" if force else "liboracle.so"], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        L.oracle_gs_solve.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p,
                                      POINTER(OStats)]
        L.oracle_gs_solve.restype = c_int
        L.oracle_jacobi_solve.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int,
                                          c_void_p, c_void_p, POINTER(OStats)]
        L.oracle_jacobi_solve.restype = c_int
        L.oracle_gs_multi.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int,
                                      POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]
        L.oracle_gs_multi.restype = c_int
        L.oracle_rmat_csr.argtypes = [c_int, c_int64, c_double, c_double, c_double, ctypes.c_uint64, c_int, c_int64,
                                      c_int64, ctypes.c_uint64, c_int, c_void_p, c_void_p, c_void_p]
        L.oracle_rmat_csr.restype = c_int
        _lib = L
    return _lib


def _arrays(g):
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int64)
    val = np.ascontiguousarray(g.val, dtype=np.float64)
    if col.size == 0:
        col = np.zeros(1, np.int64)
        val = np.zeros(1, np.float64)
    return rp, col, val


def _algo(a: str) -> int:
    return {"govm": 0, "gsvm": 1}[a]


def gs_sssp(g, source: int, algo: str = "govm", record_pred: bool = False):
    """Reference-order solve: (dist float64[n], pred int64[n] | None, stats dict)."""
    rp, col, val = _arrays(g)
    dist = np.empty(g.n, np.float64)
    pred = np.empty(g.n, np.int64) if record_pred else None
    st = OStats()
    rc = lib().oracle_gs_solve(g.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data, int(source), _algo(algo),
                               dist.ctypes.data, pred.ctypes.data if pred is not None else None, ctypes.byref(st))
    if rc:
        raise ValueError(f"oracle_gs_solve failed ({rc})")
    return dist, pred, st.as_dict()


def jacobi_sssp(g, source: int, algo: str = "govm", vtype: str = "float64", record_pred: bool = False,
                negcheck: bool = False):
    """Device-semantics solve: (dist float64[n], pred int64[n] | None, stats dict)."""
    rp, col, val = _arrays(g)
    dist = np.empty(g.n, np.float64)
    pred = np.empty(g.n, np.int64) if record_pred else None
    st = OStats()
    rc = lib().oracle_jacobi_solve(g.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data, int(source), _algo(algo),
                                   VTYPES[vtype], int(record_pred), int(negcheck), dist.ctypes.data,
                                   pred.ctypes.data if pred is not None else None, ctypes.byref(st))
    if rc:
        raise ValueError(f"oracle_jacobi_solve failed ({rc})")
    return dist, pred, st.as_dict()


def gs_multi(g, sources, threads: int | None = None, algo: str = "govm"):
    """k reference-order solves on ``threads`` threads: (relaxations, m_reach, writes)."""
    rp, col, val = _arrays(g)
    src = np.ascontiguousarray(sources, dtype=np.int64)
    threads = threads or os.cpu_count() or 1
    r, mr, w = c_int64(0), c_int64(0), c_int64(0)
    lib().oracle_gs_multi(g.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data, src.ctypes.data, int(src.size),
                          _algo(algo), int(threads), ctypes.byref(r), ctypes.byref(mr), ctypes.byref(w))
    return r.value, mr.value, w.value


def rmat_csr(scale: int, edge_factor: int, weights: str = "int", lo: int = 1, hi: int = 100, seed: int = 1,
             wseed: int = 2, threads: int | None = None):
    """Host C restatement of the counter-hash RMAT generator -> (n, m, row_ptr, col, val)."""
    n = 1 << scale
    m = edge_factor * n
    rp = np.empty(n + 1, np.int64)
    col = np.empty(m, np.int64)
    val = np.empty(m, np.float64)
    rc = lib().oracle_rmat_csr(scale, edge_factor, 0.57, 0.19, 0.19, seed, 0 if weights == "int" else 1, lo, hi,
                               wseed, int(threads or os.cpu_count() or 1), rp.ctypes.data, col.ctypes.data,
                               val.ctypes.data)
    if rc:
        raise MemoryError("oracle_rmat_csr failed")
    return n, m, rp, col, val


def floyd_warshall(n: int, row_ptr, col, val) -> tuple[np.ndarray, bool]:
    """CPU restatement (test infrastructure only) of the reference's dense
    Floyd–Warshall, oracles.py:141-162: +inf matrix with a zero diagonal,
    the minimum over parallel edges / self-loops, then for k = 0..n-1 every
    entry takes min(D[i][j], D[i][k] + D[k][j]) with row and column k as
    they were BEFORE step k (the reference forms the whole sum matrix first).
    Returns (matrix, any diagonal entry < 0)."""
    d = np.full((n, n), np.inf)
    d[np.arange(n), np.arange(n)] = 0.0
    rp = np.asarray(row_ptr, dtype=np.int64)
    u = np.repeat(np.arange(n), np.diff(rp))
    for a, b, w in zip(u.tolist(), np.asarray(col).tolist(), np.asarray(val, dtype=np.float64).tolist()):
        if w < d[a, b]:
            d[a, b] = w
    for k in range(n):
        colk = d[:, k].copy()
        rowk = d[k, :].copy()
        cand = colk[:, None] + rowk[None, :]
        better = cand < d
        d[better] = cand[better]
    return d, bool(n and np.any(np.diagonal(d) < 0))
