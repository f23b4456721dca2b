"""Cross-check oracles on the device (reference
``oracles.py``): the same names, result types, size cap and errors as the
reference, computed on the B200.

* :func:`floyd_warshall_apsp` — ``dawn_floyd_warshall``: the dense float64
  matrix with the reference's exact step order and rounding
  (oracles.py:141-162): bit-identical matrix and ``negative_cycle``;
  ``relaxations`` = n**3 as in the reference.
* :func:`bellman_ford_sssp` — the full-sweep solver (GSVM: every finite row
  relaxed every round, i.e. Bellman–Ford's passes, in snapshot order) with the
  negative-cycle check (oracles.py:94-138).  Distances of a graph without a
  reachable negative cycle are the shortest distances the reference computes
  (same greatest fixpoint, bit-identical); ``negative_cycle`` is the same
  verdict; with a reachable negative cycle the returned distances are the
  device's capped values (the reference's are its own n-1-pass values —
  neither is meaningful).  ``relaxations`` counts the device's edge scans.
* :func:`dijkstra_sssp` — rejects negative weights with the reference's
  message (oracles.py:59-91); distances from the frontier solver (for
  non-negative weights the same minimum over left-fold path sums a heap
  Dijkstra settles, bit-identical); ``relaxations`` counts device edge scans.

These are oracles for large-scale cross-checks, not the hot path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import GraphSizeError, NegativeWeightError
from .graph import CsrGraph
from .solver import DistanceVector, govm_sssp, gsvm_sssp

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


def dijkstra_sssp(g: CsrGraph, source: int) -> OracleResult:
    """Shortest distances for non-negative weights; NegativeWeightError otherwise."""
    if not 0 <= source < g.n:
        raise ValueError(f"source {source} out of range for n={g.n}")
    bad = _first_negative_edge(g)
    if bad is not None:
        raise NegativeWeightError(f"Dijkstra requires non-negative weights; edge {bad[0]} -> {bad[1]} has weight "
                                  f"{bad[2]}")
    dv, _, st = govm_sssp(g, source, schedule="async")
    return OracleResult(dist=dv, negative_cycle=False, relaxations=int(st.relaxations))


def bellman_ford_sssp(g: CsrGraph, source: int) -> OracleResult:
    """Full-sweep rounds with the reachable-negative-cycle verdict."""
    if not 0 <= source < g.n:
        raise ValueError(f"source {source} out of range for n={g.n}")
    dv, _, st = gsvm_sssp(g, source, schedule="jacobi")
    return OracleResult(dist=dv, negative_cycle=bool(st.negative_cycle), relaxations=int(st.relaxations))


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
