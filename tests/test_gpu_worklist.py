"""The barrier-free worklist tail of the async schedule (tuning key
"worklist_edges"): once a round relaxes fewer edges than the threshold the
rest of the solve runs off a ring of row items.  Distances, negative_cycle and
first_discoveries must equal the Jacobi schedule / oracle / reference for every
threshold: 0 (off), the default, and "always" (from round 2 on)."""

from __future__ import annotations

import numpy as np
import pytest
from conftest import golden_dist, golden_graph, golden_index, golden_names, make_csr

import paper_2306_07872_b200 as P
from oracle import oracle as O
from paper_2306_07872_b200 import generators as G

pytestmark = pytest.mark.gpu

DEFAULT = float(1 << 20)


@pytest.fixture(params=[0.0, DEFAULT, 1e18], ids=["off", "default", "always"])
def wl(request):
    P.set_tuning(worklist_edges=request.param, small_graph=0)  # the worklist lives in the persistent kernels
    yield request.param
    P.set_tuning(worklist_edges=DEFAULT, small_graph=-1)


def same(a, b) -> bool:
    return np.array_equal(np.asarray(a), np.asarray(b))


def check(g, src, precision="auto", algo="govm"):
    dj, _, sj = P.SOLVERS[algo](g, src, precision=precision, schedule="jacobi")
    da, _, sa = P.SOLVERS[algo](g, src, precision=precision, schedule="async")
    assert same(da.dist, dj.dist)
    assert sa.first_discoveries == sj.first_discoveries
    assert sa.negative_cycle == sj.negative_cycle
    assert sa.writes >= sa.first_discoveries
    return da, sa


@pytest.mark.parametrize("name", [n for n in golden_names() if not golden_index()[n]["stats"]["negative_cycle"]])
def test_worklist_golden(gpu, wl, name):
    meta = golden_index()[name]
    g = golden_graph(name)
    dv, _, st = P.SOLVERS[meta["algo"]](g, meta["source"], schedule="async")
    assert same(dv.dist, golden_dist(name))
    assert st.first_discoveries == meta["stats"]["first_discoveries"]


@pytest.mark.parametrize("seed", range(12))
def test_worklist_random(gpu, wl, seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(2, 3000))
    m = int(rng.integers(0, 10 * n))
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    w = [rng.integers(0, 30, m).astype(float), rng.uniform(0, 2, m),
         rng.uniform(0, 1, m).astype(np.float32).astype(float)][seed % 3]
    g = P.csr_from_arrays(n, u, v, w)
    src = int(rng.integers(0, n))
    for precision in ("auto", "fp32", "fp64"):
        da, _ = check(g, src, precision)
        vt = {"fp32": "float32", "fp64": "float64"}.get(precision) or (
            "int32" if np.all(w == np.floor(w)) else "float64")
        od, _, _ = O.jacobi_sssp(g, src, "govm", vtype=vt)
        assert same(da.dist, od)


def test_worklist_long_rows(gpu, wl):
    """Rows far longer than a chunk (448 / 256 edges): split items, chunks
    taken by different warps, the hub lowered again after its chunks ran."""
    rng = np.random.default_rng(7)
    n = 5000
    edges = []
    for hub in (1, 2, 3):
        tgt = rng.choice(n, size=4000, replace=False)
        edges += [(hub, int(t), float(rng.integers(1, 1000))) for t in tgt]
    # chains that reach the hubs late and with decreasing distances
    edges += [(0, 1, 500.0), (0, 10, 1.0), (10, 11, 1.0), (11, 1, 1.0), (0, 2, 50.0), (11, 2, 100.0)]
    edges += [(0, 20, 2.0), (20, 3, 300.0), (20, 21, 1.0), (21, 22, 1.0), (22, 3, 1.0)]
    u = rng.integers(0, n, 20000)
    v = rng.integers(0, n, 20000)
    edges += [(int(a), int(b), float(c)) for a, b, c in zip(u, v, rng.integers(1, 50, 20000))]
    g = make_csr(n, edges)
    for precision in ("auto", "fp32", "fp64"):
        da, _ = check(g, 0, precision)
        gd, _, _ = O.gs_sssp(g, 0)
        if precision != "fp32":
            assert same(da.dist, gd)


def test_worklist_zero_weights_and_unreachable(gpu, wl):
    g = make_csr(8, [(0, 1, 0.0), (1, 2, 0.0), (2, 0, 0.0), (2, 3, 1.0), (5, 6, 1.0), (3, 3, 0.0)])
    da, sa = check(g, 0)
    assert same(da.dist, [0, 0, 0, 1, np.inf, np.inf, np.inf, np.inf])
    assert sa.first_discoveries == 3
    e = make_csr(4, [])
    da, sa = check(e, 2)
    assert sa.first_discoveries == 0


def test_worklist_rmat_and_grid(gpu, wl):
    g = G.rmat_graph(17, 16, weights="f32")
    for _ in range(2):
        check(g, 0, "fp32")
    gi = G.rmat_graph(15, 8, weights="int")
    da, _ = check(gi, 3)
    assert same(da.dist, O.gs_sssp(gi, 3)[0])
    grid = G.grid_graph(96, 80)
    P.set_tuning(bitmap_frontier=0)  # the worklist lives in the queue-frontier kernels
    try:
        da, _ = check(grid, 0)
        assert same(da.dist, O.gs_sssp(grid, 0)[0])
    finally:
        P.set_tuning(bitmap_frontier=-1)


def test_worklist_not_used_when_stepping(gpu):
    """trace= steps round by round: the worklist must not take over."""
    P.set_tuning(worklist_edges=1e18)
    try:
        g = golden_graph(golden_names("rnd_uniform02_")[0])
        records = []
        dv, _, st = P.govm_sssp(g, 0, trace=lambda *a: records.append(a), schedule="async")
        assert records
        prev = None
        for step, scanned, written, alpha in records:
            if prev is not None:
                assert scanned == prev
            prev = written
        assert same(dv.dist, P.govm_sssp(g, 0)[0].dist)
    finally:
        P.set_tuning(worklist_edges=DEFAULT)


def test_worklist_long_chain(gpu):
    """A 20 000-hop dependency chain (8 parallel edges per hop, so the queue
    frontier and the tail are used, not the bitmap frontier): the worklist runs
    a long serial chain of local batches while every other warp waits."""
    n = 20000
    rng = np.random.default_rng(3)
    u = np.repeat(np.arange(n - 1), 8)
    v = u + 1
    w = rng.integers(1, 9, u.size).astype(float)
    # a few long-range shortcuts with large weights (never on the shortest path)
    su = rng.integers(0, n, 2000)
    sv = rng.integers(0, n, 2000)
    g = P.csr_from_arrays(n, np.concatenate([u, su]), np.concatenate([v, sv]),
                          np.concatenate([w, np.full(2000, 1e6)]))
    da, _, sa = P.govm_sssp(g, 0, schedule="async")
    od, _, _ = O.gs_sssp(g, 0)
    assert same(da.dist, od)
