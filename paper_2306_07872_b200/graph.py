"""Host-side graph containers: the input contract of the hot path.

``CsrGraph`` is the reference's immutable CSR type (graph.py:64-109 of
``sparsepath``): int64 ``row_ptr[n+1]``, int64 ``col[m]``, float64 ``val[m]``,
rows sorted by destination with ties in input order, arrays read-only.  The
solvers in this package accept it (or the reference's own ``CsrGraph``, or
any object with the same five attributes) and upload it once to the device
(``DeviceGraph``, cached per graph object).

``EdgeList``/``build_csr``/``WeightMode``/``apply_weight_mode``/
``generate_random_graph`` are thin numpy helpers kept API-compatible so
callers and tests can build inputs; file I/O is out of scope.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "EdgeList",
    "CsrGraph",
    "WeightMode",
    "build_csr",
    "to_edge_list",
    "apply_weight_mode",
    "generate_random_graph",
]


@dataclass
class EdgeList:
    """Directed edges ``(u, v, w)`` before CSR construction (reference graph.py:43-61).

    Duplicates and self-loops are allowed; ``n`` may exceed the largest id.
    """

    n: int
    edges: list[tuple[int, int, float]] = field(default_factory=list)

    def validate(self) -> None:
        if self.n < 0:
            raise ValueError(f"node count must be non-negative, got {self.n}")
        n = self.n
        for u, v, w in self.edges:
            if u < 0 or v < 0 or u >= n or v >= n:
                raise ValueError(f"edge ({u}, {v}) out of range for n={n}")
            if not math.isfinite(w):
                raise ValueError(f"edge ({u}, {v}) has non-finite weight {w!r}")


@dataclass(frozen=True, eq=False)
class CsrGraph:
    """Immutable CSR adjacency with float64 weights (reference graph.py:64-109).

    Out-edges of ``u`` are ``col[row_ptr[u]:row_ptr[u+1]]`` / ``val[...]``.
    Identity-hashed (``eq=False``), which is what the device-upload cache keys on.
    """

    n: int
    m: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    def __post_init__(self):
        rp = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(self.col, dtype=np.int64)
        val = np.ascontiguousarray(self.val, dtype=np.float64)
        for name, arr in (("row_ptr", rp), ("col", col), ("val", val)):
            object.__setattr__(self, name, arr)
        n, m = self.n, self.m
        if n < 0:
            raise ValueError("node count must be non-negative")
        if rp.shape != (n + 1,):
            raise ValueError("row_ptr must have length n + 1")
        if rp[0] != 0 or rp[-1] != m:
            raise ValueError("row_ptr must start at 0 and end at m")
        if n and (np.diff(rp) < 0).any():
            raise ValueError("row_ptr must be monotone non-decreasing")
        if col.shape != (m,) or val.shape != (m,):
            raise ValueError("col and val must both have length m")
        if m:
            if col.min() < 0 or col.max() >= n:
                raise ValueError("column index out of range")
            if not np.isfinite(val).all():
                raise ValueError("weights must be finite")
        for arr in (rp, col, val):
            arr.flags.writeable = False

    def out_degree(self, u: int) -> int:
        return int(self.row_ptr[u + 1]) - int(self.row_ptr[u])


def csr_from_arrays(n: int, u: np.ndarray, v: np.ndarray, w: np.ndarray) -> CsrGraph:
    """Canonical CSR from parallel edge arrays: rows by source, then by
    destination, ties in input order (the ordering of reference graph.py:303-322)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    m = int(u.shape[0])
    if m == 0:
        return CsrGraph(n, 0, np.zeros(n + 1, np.int64), np.empty(0, np.int64), np.empty(0, np.float64))
    if n <= (1 << 31):
        order = np.argsort(u * n + v, kind="stable")
    else:
        order = np.lexsort((v, u))
    counts = np.bincount(u, minlength=n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    return CsrGraph(n=n, m=m, row_ptr=rp, col=v[order], val=w[order])


def build_csr(el: EdgeList) -> CsrGraph:
    """CSR of an ``EdgeList`` in canonical order, duplicates kept."""
    el.validate()
    m = len(el.edges)
    if m == 0:
        return csr_from_arrays(el.n, np.empty(0), np.empty(0), np.empty(0))
    arr = np.array([(e[0], e[1]) for e in el.edges], dtype=np.int64).reshape(m, 2)
    w = np.fromiter((e[2] for e in el.edges), dtype=np.float64, count=m)
    return csr_from_arrays(el.n, arr[:, 0], arr[:, 1], w)


def to_edge_list(g) -> EdgeList:
    """Row-major edge list of a CSR graph (rebuilding it gives the same arrays)."""
    rp = np.asarray(g.row_ptr)
    u = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(rp))
    return EdgeList(n=g.n, edges=list(zip(u.tolist(), np.asarray(g.col).tolist(), np.asarray(g.val).tolist())))


@dataclass(frozen=True)
class WeightMode:
    """Weight assignment: keep, unit, or seeded uniform ``[lo, hi)`` (reference graph.py:112-142)."""

    kind: str
    lo: float = 0.0
    hi: float = 0.0
    seed: int = 0

    KEEP = "keep"
    UNIT = "unit"
    RANDOM = "random"

    @classmethod
    def keep(cls) -> "WeightMode":
        return cls(cls.KEEP)

    @classmethod
    def unit(cls) -> "WeightMode":
        return cls(cls.UNIT)

    @classmethod
    def random_uniform(cls, lo: float, hi: float, seed: int) -> "WeightMode":
        if not lo < hi:
            raise ValueError(f"invalid weight range [{lo}, {hi}): lo must be < hi")
        return cls(cls.RANDOM, lo=lo, hi=hi, seed=seed)


def apply_weight_mode(g: CsrGraph, mode: WeightMode) -> CsrGraph:
    """Same structure, new weights."""
    if mode.kind == WeightMode.KEEP:
        return g
    if mode.kind == WeightMode.UNIT:
        val = np.ones(g.m)
    elif mode.kind == WeightMode.RANDOM:
        if not mode.lo < mode.hi:
            raise ValueError(f"invalid weight range [{mode.lo}, {mode.hi})")
        val = np.random.default_rng(mode.seed).uniform(mode.lo, mode.hi, size=g.m)
    else:
        raise ValueError(f"unknown weight mode {mode.kind!r}")
    return CsrGraph(n=g.n, m=g.m, row_ptr=g.row_ptr, col=g.col, val=val)


def generate_random_graph(n: int, avg_degree: float, mode: WeightMode, seed: int) -> CsrGraph:
    """Seeded directed Erdos-Renyi graph without self-loops or duplicate edges.

    Every ordered pair ``u != v`` is present with probability
    ``avg_degree / (n - 1)``; base weights are 1.0 before ``mode`` applies.
    """
    if n < 0:
        raise ValueError("n must be non-negative")
    if avg_degree < 0:
        raise ValueError("avg_degree must be non-negative")
    if n == 0:
        return build_csr(EdgeList(n=0))
    p = avg_degree / max(n - 1, 1)
    if p > 1.0:
        warnings.warn(f"avg_degree {avg_degree} exceeds n-1={n - 1}; clamping edge probability to 1", stacklevel=2)
        p = 1.0
    rng = np.random.default_rng(seed)
    us, vs = [], []
    for u in range(n):
        k = int(rng.binomial(n - 1, p)) if n > 1 else 0
        if k == 0:
            continue
        # k distinct targets among the n-1 non-self slots, drawn exactly as the
        # reference does (graph.py:433-443): batches of 2*(missing) uniform
        # slot draws until k distinct ones are in; the set is sorted
        chosen: set[int] = set()
        while len(chosen) < k:
            for t in rng.integers(0, n - 1, size=2 * (k - len(chosen))).tolist():
                chosen.add(t + 1 if t >= u else t)
                if len(chosen) == k:
                    break
        us.append(np.full(k, u, np.int64))
        vs.append(np.array(sorted(chosen), dtype=np.int64))
    if us:
        u_arr, v_arr = np.concatenate(us), np.concatenate(vs)
    else:
        u_arr = v_arr = np.empty(0, np.int64)
    g = csr_from_arrays(n, u_arr, v_arr, np.ones(u_arr.shape[0]))
    return apply_weight_mode(g, mode)
