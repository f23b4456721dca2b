"""Synthetic inputs for the BASELINE configurations.

All randomness comes from one counter-based hash so the host restatement
here and the device generator (``dawn_gen_rmat`` in csrc/dawn.cu) produce the
SAME graph bit for bit:

    mix64(z)        = splitmix64 finaliser
    draw(seed,i,l)  = mix64(seed*G + i*64 + l + G)  (mod 2^64), G = 0x9E3779B97F4A7C15

* RMAT (Graph500 a,b,c = .57,.19,.19): edge i, level l (bit l, LSB first)
  takes q = draw(seed,i,l) >> 40 (24 bits); q <  A -> (0,0); q < AB -> (0,1);
  q < ABC -> (1,0); else (1,1), with A = floor(a*2^24) etc.  No relabelling,
  so vertex 0 is the hub and "source 0" is meaningful; duplicates and
  self-loops are kept (as the reference's build_csr keeps them).
* Weights of edge i use h = draw(wseed, i, 63): integers
  ``lo + ((h>>32) * (hi-lo+1)) >> 32``, or float32 ``(h>>40) * 2^-24`` in [0,1).
* Grid: r x c 4-neighbour lattice, both directions, edge order = CSR order.
* Johnson potentials p[v] = lo + (draw(pseed, v, 62)>>32)*range>>32 turn base
  weights w into w + p[u] - p[v]: negative edges, no negative cycle.
* Injected cycles follow the reference test generator's recipe
  (tests/_gen.py:47-69): length 2-4, positive edges, closing edge
  -(sum + 5), plus an edge source -> cycle[0].
"""

from __future__ import annotations

import numpy as np

from .graph import CsrGraph, csr_from_arrays

G = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= M1
    z ^= z >> np.uint64(27)
    z *= M2
    z ^= z >> np.uint64(31)
    return z


def draw(seed: int, idx: np.ndarray, level: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * G + np.uint64(level) + G
        return mix64(idx.astype(np.uint64) * np.uint64(64) + base)


def _weights(m: int, wseed: int, kind: str, lo: int, hi: int, chunk: int = 1 << 24) -> np.ndarray:
    out = np.empty(m, dtype=np.float64)
    for s in range(0, m, chunk):
        idx = np.arange(s, min(m, s + chunk), dtype=np.uint64)
        h = draw(wseed, idx, 63)
        if kind == "int":
            rng = np.uint64(hi - lo + 1)
            out[s:s + idx.size] = lo + (((h >> np.uint64(32)) * rng) >> np.uint64(32)).astype(np.int64)
        else:
            out[s:s + idx.size] = ((h >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)).astype(np.float64)
    return out


def rmat_edges(scale: int, edge_factor: int, seed: int = 1, a: float = 0.57, b: float = 0.19, c: float = 0.19,
               chunk: int = 1 << 22):
    """Host restatement of ``dawn_gen_rmat``: (u, v) int64 arrays of m = ef * 2^scale edges."""
    n = 1 << scale
    m = edge_factor * n
    A, AB, ABC = (np.uint64(int(x * 16777216.0)) for x in (a, a + b, a + b + c))
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for s in range(0, m, chunk):
        idx = np.arange(s, min(m, s + chunk), dtype=np.uint64)
        uu = np.zeros(idx.size, dtype=np.int64)
        vv = np.zeros(idx.size, dtype=np.int64)
        for lvl in range(scale):
            q = draw(seed, idx, lvl) >> np.uint64(40)
            ub = q >= AB
            vb = ((q >= A) & (q < AB)) | (q >= ABC)
            uu |= ub.astype(np.int64) << lvl
            vv |= vb.astype(np.int64) << lvl
        u[s:s + idx.size] = uu
        v[s:s + idx.size] = vv
    return n, u, v


def rmat_graph(scale: int, edge_factor: int, weights: str = "int", lo: int = 1, hi: int = 100, seed: int = 1,
               wseed: int = 2) -> CsrGraph:
    """RMAT CsrGraph; ``weights`` = "int" (uniform [lo, hi]) or "f32" (float32 in [0,1))."""
    n, u, v = rmat_edges(scale, edge_factor, seed)
    w = _weights(u.size, wseed, "int" if weights == "int" else "f32", lo, hi)
    return csr_from_arrays(n, u, v, w)


def grid_graph(rows: int, cols: int, lo: int = 1, hi: int = 100, wseed: int = 2) -> CsrGraph:
    """4-neighbour grid, both directions, integer weights; node id = r*cols + c."""
    n = rows * cols
    ids = np.arange(n, dtype=np.int64)
    r, c = ids // cols, ids % cols
    nbrs = []
    for dr, dc in ((-1, 0), (0, -1), (0, 1), (1, 0)):  # ascending neighbour id
        ok = (r + dr >= 0) & (r + dr < rows) & (c + dc >= 0) & (c + dc < cols)
        nbrs.append(np.where(ok, ids + dr * cols + dc, -1))
    nb = np.stack(nbrs, axis=1)  # [n, 4]
    mask = nb >= 0
    deg = mask.sum(axis=1)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = nb[mask]
    w = _weights(col.size, wseed, "int", lo, hi)
    return CsrGraph(n=n, m=int(col.size), row_ptr=rp, col=col, val=w)


def johnson_reweight(g: CsrGraph, pseed: int = 3, lo: int = 0, hi: int = 199) -> tuple[CsrGraph, np.ndarray]:
    """w'(u,v) = w + p[u] - p[v]: negative edges without negative cycles."""
    idx = np.arange(g.n, dtype=np.uint64)
    h = draw(pseed, idx, 62)
    p = lo + (((h >> np.uint64(32)) * np.uint64(hi - lo + 1)) >> np.uint64(32)).astype(np.int64)
    u = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
    val = g.val + p[u] - p[g.col]
    return CsrGraph(n=g.n, m=g.m, row_ptr=g.row_ptr, col=g.col, val=val), p


def inject_cycles(g: CsrGraph, k: int, source: int = 0, seed: int = 4, reachable: bool = True) -> CsrGraph:
    """Add ``k`` negative cycles (length 2-4, closing edge -(sum+5)); if
    ``reachable`` also add source -> cycle[0] (weight 1)."""
    rng = np.random.default_rng(seed)
    pool = np.arange(g.n)
    if not reachable:
        # nodes nobody points at stay unreachable once only the cycle feeds them
        indeg = np.bincount(g.col, minlength=g.n)
        pool = np.flatnonzero((indeg == 0) & (np.arange(g.n) != source))
        if pool.size < 4 * k:
            raise ValueError("not enough in-degree-0 nodes for unreachable cycles")
        pool = rng.permutation(pool)[: 4 * k]
    us, vs, ws = [], [], []
    for ci in range(k):
        length = int(rng.integers(2, 5))
        if reachable:
            cyc = [int(x) for x in rng.choice(g.n, size=length, replace=False)]
        else:
            cyc = [int(x) for x in pool[4 * ci: 4 * ci + length]]
        total = 0
        for a_, b_ in zip(cyc, cyc[1:]):
            w = int(rng.integers(1, 101))
            total += w
            us.append(a_); vs.append(b_); ws.append(float(w))
        us.append(cyc[-1]); vs.append(cyc[0]); ws.append(float(-(total + 5)))
        if reachable:
            us.append(source); vs.append(cyc[0]); ws.append(1.0)
    u0 = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
    u = np.concatenate([u0, np.asarray(us, np.int64)])
    v = np.concatenate([g.col, np.asarray(vs, np.int64)])
    w = np.concatenate([g.val, np.asarray(ws, np.float64)])
    return csr_from_arrays(g.n, u, v, w)
