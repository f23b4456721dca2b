"""The near-far schedule (dawn_nearfar.cuh): async solves on graphs without
negative weights, relaxed in bucket order from a pending-row bitmap with
per-warp continuation rings.  Distances, first_discoveries and the
negative-cycle flag (always False here) must equal the Jacobi oracle /
reference exactly, for every bucket width; the work counters are the run's
own and only bounded."""

from __future__ import annotations

import numpy as np
import pytest
from conftest import golden_dist, golden_graph, golden_index, golden_names

import paper_2306_07872_b200 as P
from oracle import oracle as O
from paper_2306_07872_b200 import generators as G

pytestmark = pytest.mark.gpu


def same(a, b) -> bool:
    return np.array_equal(np.asarray(a), np.asarray(b))


@pytest.fixture
def nearfar():
    """Force the near-far path (auto enables it only on low-degree graphs with n >= 4096)."""
    P.set_tuning(nearfar=1, small_graph=0)
    yield
    P.set_tuning(nearfar=-1, nearfar_delta=0, nearfar_delta_mean=8, small_graph=-1)


def _vtype(w, precision):
    if precision == "fp32":
        return "float32"
    if precision == "fp64":
        return "float64"
    return "int32" if np.all(w == np.floor(w)) else "float64"


def _nonneg_golden():
    out = []
    for name in golden_names():
        meta = golden_index()[name]
        if meta["algo"] == "govm" and not meta["stats"]["negative_cycle"]:
            g = golden_graph(name)
            if g.m == 0 or float(np.min(g.val)) >= 0:
                out.append(name)
    return out


@pytest.mark.parametrize("name", _nonneg_golden())
def test_nearfar_golden(gpu, nearfar, name):
    meta = golden_index()[name]
    g = golden_graph(name)
    dv, _, st = P.govm_sssp(g, meta["source"], schedule="async")
    assert same(dv.dist, golden_dist(name))
    assert st.first_discoveries == meta["stats"]["first_discoveries"]
    assert not st.negative_cycle
    assert st.writes >= st.first_discoveries


@pytest.mark.parametrize("seed", range(24))
def test_nearfar_random_vs_oracle(gpu, nearfar, seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(0, 6 * n))
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    w = [rng.integers(1, 50, m).astype(float), rng.uniform(0, 2, m),
         rng.uniform(0, 1, m).astype(np.float32).astype(float), rng.integers(0, 3, m).astype(float)][seed % 4]
    g = P.csr_from_arrays(n, u, v, w)
    src = int(rng.integers(0, n))
    # bucket widths from "one value per bucket" to "everything near"
    P.set_tuning(nearfar_delta=[0, 0.01, 1.0, 1e9][seed // 4 % 4])
    for precision in ("auto", "fp32", "fp64"):
        dv, _, st = P.govm_sssp(g, src, precision=precision, schedule="async")
        od, _, o = O.jacobi_sssp(g, src, "govm", vtype=_vtype(w, precision))
        assert same(dv.dist, od), precision
        assert st.first_discoveries == o["first_discoveries"]
        assert not st.negative_cycle
        assert st.writes >= st.first_discoveries and st.relaxations >= 0


@pytest.mark.parametrize("side,delta", [(64, 0), (200, 1), (200, 0), (333, 5000), (512, 0)])
def test_nearfar_grid_vs_oracle(gpu, side, delta):
    """Grids take the near-far path by default (low degree, n >= 4096)."""
    g = G.grid_graph(side, side)
    P.set_tuning(nearfar_delta=delta)
    try:
        for src in (0, g.n // 2 + side // 3, g.n - 1):
            dv, _, st = P.govm_sssp(g, src, schedule="async")
            od, _, o = O.jacobi_sssp(g, src, "govm", vtype="int32")
            assert same(dv.dist, od)
            assert st.first_discoveries == o["first_discoveries"]
            if delta == 0 and side >= 200:  # bucket order: far fewer relaxations than the snapshot rounds
                assert st.relaxations < o["relaxations"] / 2
    finally:
        P.set_tuning(nearfar_delta=0)


def test_nearfar_chain_star_and_isolated(gpu, nearfar):
    # a long path: the whole chain runs inside one warp's ring
    n = 20000
    g = P.csr_from_arrays(n, np.arange(n - 1), np.arange(1, n), np.full(n - 1, 3.0))
    dv, _, st = P.govm_sssp(g, 0, schedule="async")
    assert same(dv.dist, 3.0 * np.arange(n)) and st.first_discoveries == n - 1
    # a star with a 50k-edge row (warp-cooperative expansion of a long row) and duplicate edges
    hub = 50000
    rng = np.random.default_rng(3)
    u = np.concatenate([np.zeros(hub, np.int64), rng.integers(1, hub, 20000)])
    v = np.concatenate([rng.integers(1, hub, hub), rng.integers(1, hub, 20000)])
    w = rng.integers(1, 1000, u.size).astype(float)
    g = P.csr_from_arrays(hub, u, v, w)
    dv, _, _ = P.govm_sssp(g, 0, schedule="async")
    assert same(dv.dist, O.jacobi_sssp(g, 0, "govm", vtype="int32")[0])
    # isolated source, single node
    g = P.csr_from_arrays(5, np.array([1]), np.array([2]), np.array([1.0]))
    dv, _, st = P.govm_sssp(g, 0, schedule="async")
    assert dv.dist.tolist() == [0.0, np.inf, np.inf, np.inf, np.inf] and st.first_discoveries == 0
    g1 = P.csr_from_arrays(1, np.array([], np.int64), np.array([], np.int64), np.array([]))
    assert P.govm_sssp(g1, 0, schedule="async")[0].dist.tolist() == [0.0]


def test_nearfar_repeatable_and_mixed_with_jacobi(gpu):
    """Same solver object alternating schedules; the near-far run leaves no
    pending bits behind for the next solve."""
    g = G.grid_graph(300, 300)
    od, _, o = O.jacobi_sssp(g, 7, "govm", vtype="int32")
    for _ in range(3):
        da, _, sa = P.govm_sssp(g, 7, schedule="async")
        dj, _, sj = P.govm_sssp(g, 7, schedule="jacobi")
        assert same(da.dist, od) and same(dj.dist, od)
        assert (sj.relaxations, sj.writes, sj.outer_steps) == (o["relaxations"], o["writes"], o["outer_steps"])


def test_nearfar_not_used_with_negative_weights_or_pred(gpu, nearfar):
    base, _ = G.johnson_reweight(G.rmat_graph(11, 4), pseed=3)
    da, _, sa = P.govm_sssp(base, 0, schedule="async")
    dj, _, sj = P.govm_sssp(base, 0)
    assert same(da.dist, dj.dist) and sa.as_dict() == sj.as_dict()
    g = G.grid_graph(100, 100)
    dv, pv, _ = P.govm_sssp(g, 0, record_pred=True, schedule="async")
    assert same(dv.dist, O.jacobi_sssp(g, 0, "govm", vtype="int32")[0])
    assert pv.path_to(g.n - 1)[0] == 0
