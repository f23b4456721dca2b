"""Cross-check oracles on the device (reference
``oracles.py``): the same names, result types, size cap and errors as the
reference, computed on the B200.

* :func:`floyd_warshall_apsp` — ``dawn_floyd_warshall``: the dense float64
  matrix with the reference's exact step order and rounding
  (oracles.py:141-162): bit-identical matrix and ``negative_cycle``;
  ``relaxations`` = n**3 as in the reference.
* :func:`dijkstra_sssp` / :func:`bellman_ford_sssp` — independent of the
  device kernels on purpose (they exist to check them; computing them with the
  solvers under test would make every cross-check circular): native host
  restatements in libdawn (``dawn_oracle_dijkstra`` /
  ``dawn_oracle_bellman_ford``, csrc/dawn_host_oracles.cpp) of the reference's
  heap Dijkstra (oracles.py:59-91) and textbook n-1-pass Bellman–Ford with its
  detection pass (oracles.py:94-138).  Same visiting order and float64
  arithmetic, so distances, ``relaxations`` and ``negative_cycle`` equal the
  reference's exactly — including its unguarded distances on a reachable
  negative cycle.

These are oracles for large-scale cross-checks, not the hot path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import GraphSizeError, NegativeWeightError
from .graph import CsrGraph
from .solver import DistanceVector

__all__ = ["OracleResult", "FloydResult", "dijkstra_sssp", "bellman_ford_sssp", "floyd_warshall_apsp",
           "DEFAULT_FLOYD_CAP"]

DEFAULT_FLOYD_CAP = 2000  # oracles.py:32


@dataclass
class OracleResult:
    dist: DistanceVector
    negative_cycle: bool
    relaxations: int


@dataclass
class FloydResult:
    matrix: np.ndarray
    negative_cycle: bool
    relaxations: int


def _first_negative_edge(g: CsrGraph):
    """(u, v, w) of the smallest weight if it is negative (the edge the reference names)."""
    if g.m == 0:
        return None
    k = int(np.argmin(g.val))
    if g.val[k] >= 0:
        return None
    u = int(np.searchsorted(g.row_ptr, k, side="right")) - 1
    return u, int(g.col[k]), float(g.val[k])


def _host_arrays(g: CsrGraph):
    return (np.ascontiguousarray(g.row_ptr, dtype=np.int64), np.ascontiguousarray(g.col, dtype=np.int64),
            np.ascontiguousarray(g.val, dtype=np.float64))


def dijkstra_sssp(g: CsrGraph, source: int) -> OracleResult:
    """Heap Dijkstra (oracles.py:59-91); NegativeWeightError on a negative weight."""
    if not 0 <= source < g.n:
        raise ValueError(f"source {source} out of range for n={g.n}")
    bad = _first_negative_edge(g)
    if bad is not None:
        raise NegativeWeightError(f"Dijkstra requires non-negative weights; edge {bad[0]} -> {bad[1]} has weight "
                                  f"{bad[2]}")
    rp, col, val = _host_arrays(g)
    dist = np.empty(g.n, dtype=np.float64)
    relax = ctypes.c_int64(0)
    N.check(N.lib().dawn_oracle_dijkstra(g.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data, int(source),
                                         dist.ctypes.data, ctypes.byref(relax)))
    return OracleResult(dist=DistanceVector(dist=dist, source=int(source)), negative_cycle=False,
                        relaxations=relax.value)


def bellman_ford_sssp(g: CsrGraph, source: int) -> OracleResult:
    """Textbook Bellman–Ford with the reachable-negative-cycle verdict (oracles.py:94-138)."""
    if not 0 <= source < g.n:
        raise ValueError(f"source {source} out of range for n={g.n}")
    rp, col, val = _host_arrays(g)
    dist = np.empty(g.n, dtype=np.float64)
    relax, neg = ctypes.c_int64(0), ctypes.c_int(0)
    N.check(N.lib().dawn_oracle_bellman_ford(g.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data, int(source),
                                             dist.ctypes.data, ctypes.byref(relax), ctypes.byref(neg)))
    return OracleResult(dist=DistanceVector(dist=dist, source=int(source)), negative_cycle=bool(neg.value),
                        relaxations=relax.value)


def floyd_warshall_apsp(g: CsrGraph, cap: int = DEFAULT_FLOYD_CAP, device: int = 0) -> FloydResult:
    """Dense all-pairs matrix (n <= cap), a negative diagonal entry flags a negative cycle."""
    n = g.n
    if n > cap:
        raise GraphSizeError(f"n={n} exceeds the Floyd-Warshall cap of {cap}; run a per-source oracle "
                             "(Dijkstra or Bellman-Ford) instead")
    if n == 0:
        return FloydResult(matrix=np.zeros((0, 0)), negative_cycle=False, relaxations=0)
    N.require_gpu()
    import torch

    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int64)
    val = np.ascontiguousarray(g.val, dtype=np.float64)
    out = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
    neg = ctypes.c_int(0)
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream(device).cuda_stream
        N.check(N.lib().dawn_floyd_warshall(device, n, rp.ctypes.data, col.ctypes.data if g.m else None,
                                            val.ctypes.data if g.m else None, out.ctypes.data, ctypes.byref(neg),
                                            stream))
    return FloydResult(matrix=out, negative_cycle=bool(neg.value), relaxations=n ** 3)
