"""GPU parity of the batched multi-source kernel (dawn_mssp_batch, K9).

Every row and every per-source counter of a batched solve must equal the
single-source solve of the same source (same snapshot-Jacobi rounds per
lane) and therefore the oracle; distances equal the reference-order port."""

from __future__ import annotations

import numpy as np
import pytest
import torch
from conftest import golden_graph, make_csr

import paper_2306_07872_b200 as P
from oracle import oracle as O
from paper_2306_07872_b200 import generators as G
from paper_2306_07872_b200 import multisource as MS

pytestmark = pytest.mark.gpu


def same(a, b) -> bool:
    return np.array_equal(np.asarray(a), np.asarray(b))


def single(g, s, algo, precision=None):
    return P.SOLVERS[algo](g, s, precision=precision)


def check_rows(g, sources, algo, tile, stats, precision=None):
    t = tile.double().cpu().numpy() if isinstance(tile, torch.Tensor) else tile
    for i, s in enumerate(sources):
        dv, _, st = single(g, s, algo, precision)
        assert same(t[i, : g.n], dv.dist), (algo, i, s)
        assert stats[i].as_dict() == st.as_dict(), (algo, i, s)


@pytest.fixture(params=[4, 0, 33], ids=["auto", "dense-lanes", "sparse-lanes"])
def lane_mode(request):
    """Batched relax: default lane-sparse policy, never, always."""
    P.set_tuning(batch_sparse_util=request.param)
    yield request.param
    P.set_tuning(batch_sparse_util=4)


@pytest.mark.parametrize("seed", range(10))
def test_batch_random_vs_single(gpu, seed, lane_mode):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 600))
    m = int(rng.integers(0, 8 * n))
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    w = rng.integers(0, 40, m).astype(float) if seed % 2 == 0 else rng.uniform(0, 2, m)
    g = P.csr_from_arrays(n, u, v, w)
    k = [1, 5, 31, 32, 33, 70, 3, 64, 40, 2][seed]
    src = [int(x) for x in rng.integers(0, n, k)]
    if k > 3:
        src[1] = src[0]  # duplicate sources share a node in one batch
    for algo in ("govm", "gsvm"):
        tile, stats = MS.mssp_tile(g, src, algo)
        check_rows(g, src, algo, tile, stats)


def test_batch_is_the_mssp_path(gpu):
    g = golden_graph("rnd_uniform02_5_govm")
    rows = P.mssp(g, range(g.n), "govm")
    for s, (dv, st) in enumerate(rows):
        dv1, _, st1 = P.govm_sssp(g, s)
        assert same(dv.dist, dv1.dist) and st.as_dict() == st1.as_dict()


def test_batch_rmat14_int_vs_reference_port(gpu, lane_mode):
    g = G.rmat_graph(14, 8, weights="int")  # config 1's shape
    rng = np.random.default_rng(5)
    deg = np.diff(g.row_ptr)
    src = sorted(int(x) for x in rng.choice(np.flatnonzero(deg > 0), size=70, replace=False))
    tile, stats = MS.mssp_tile(g, src, "govm")
    t = tile.cpu().numpy()
    for i, s in enumerate(src[:12]):
        gd, _, _ = O.gs_sssp(g, s)
        assert same(t[i], gd)
        od, _, o = O.jacobi_sssp(g, s, "govm", vtype="int32")
        assert stats[i].relaxations == o["relaxations"] and stats[i].writes == o["writes"]
        assert stats[i].outer_steps == o["outer_steps"] and stats[i].first_discoveries == o["first_discoveries"]
    check_rows(g, src[12:20], "govm", t[12:20], stats[12:20])


def test_batch_fp32_tile(gpu, lane_mode):
    g = G.rmat_graph(15, 16, weights="f32")
    src = list(range(0, 2000, 31))
    tile, stats = MS.mssp_tile(g, src, "govm", precision="fp32", out_dtype=torch.float32)
    assert tile.dtype == torch.float32
    for i in (0, 7, 33, len(src) - 1):
        od, _, o = O.jacobi_sssp(g, src[i], "govm", vtype="float32")
        assert same(tile[i].double().cpu().numpy(), od)
        assert stats[i].relaxations == o["relaxations"] and stats[i].writes == o["writes"]
    # float64 tile of the same fp32 solve holds the same values
    t64, _ = MS.mssp_tile(g, src, "govm", precision="fp32")
    assert same(t64.cpu().numpy(), tile.double().cpu().numpy())


def test_batch_strided_out_and_grid(gpu):
    g = G.grid_graph(48, 40)
    src = [0, 5, 1919, 777, 1000] * 9
    big = torch.full((len(src), g.n + 17), -7.0, dtype=torch.float64, device="cuda")
    view = big[:, : g.n]
    tile, stats = MS.mssp_tile(g, src, "govm", out=view)
    assert bool((big[:, g.n:] == -7.0).all())
    check_rows(g, src[:5], "govm", tile[:5], stats[:5])
    assert all(stats[i].as_dict() == stats[i % 5].as_dict() for i in range(len(src)))


def test_batch_negative_weights_fall_back(gpu):
    base, _ = G.johnson_reweight(G.rmat_graph(10, 8), pseed=3)
    dg = P.device_graph(base)
    assert not MS.batch_supported(dg)
    src = [0, 3, 9]
    tile, stats = MS.mssp_tile(base, src, "govm")
    check_rows(base, src, "govm", tile, stats)
    cyc = G.inject_cycles(base, 1, source=0, seed=7)
    tile, stats = MS.mssp_tile(cyc, [0], "govm")
    assert stats[0].negative_cycle


def test_edgeless_and_isolated(gpu):
    e = make_csr(5, [])
    tile, stats = MS.mssp_tile(e, [0, 4, 2], "govm")
    t = tile.cpu().numpy()
    for i, s in enumerate([0, 4, 2]):
        want = np.full(5, np.inf)
        want[s] = 0
        assert same(t[i], want) and stats[i].outer_steps == 2 and stats[i].writes == 0
    g = make_csr(3, [(1, 2, 1.0)])
    tile, stats = MS.mssp_tile(g, [0, 1, 0, 1], "gsvm")
    check_rows(g, [0, 1, 0, 1], "gsvm", tile, stats)


@pytest.mark.parametrize("seed", range(8))
def test_batch_async_rows(gpu, seed, lane_mode):
    """Async batches (live distance lines instead of round-start snapshots):
    every row and first_discoveries equal the Jacobi batch / oracle."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(2, 900))
    m = int(rng.integers(0, 10 * n))
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    w = rng.integers(0, 40, m).astype(float) if seed % 2 == 0 else rng.uniform(0, 2, m)
    g = P.csr_from_arrays(n, u, v, w)
    k = [1, 5, 32, 33, 70, 64, 40, 2][seed]
    src = [int(x) for x in rng.integers(0, n, k)]
    for algo in ("govm", "gsvm"):
        tj, sj = MS.mssp_tile(g, src, algo, schedule="jacobi")
        ta, sa = MS.mssp_tile(g, src, algo, schedule="async")
        assert same(ta.cpu().numpy(), tj.cpu().numpy()), algo
        for a, b in zip(sa, sj):
            assert a.first_discoveries == b.first_discoveries and a.negative_cycle == b.negative_cycle
            assert a.writes >= a.first_discoveries


def test_batch_async_rmat_and_api(gpu):
    g = G.rmat_graph(15, 16, weights="f32")
    src = list(range(0, 3000, 37))
    tj, sj = MS.mssp_tile(g, src, "govm", precision="fp32", out_dtype=torch.float32, schedule="jacobi")
    ta, sa = MS.mssp_tile(g, src, "govm", precision="fp32", out_dtype=torch.float32, schedule="async")
    assert torch.equal(ta, tj)
    assert sum(s.relaxations for s in sa) <= sum(s.relaxations for s in sj)
    gi = G.rmat_graph(12, 8, weights="int")
    rows = P.mssp(gi, range(0, 200, 3), "govm", schedule="async")
    for s, (dv, st) in zip(range(0, 200, 3), rows):
        assert same(dv.dist, O.gs_sssp(gi, s)[0])
    got = []
    agg = P.apsp(gi, "govm", sink=got.append, schedule="async")
    assert [d.source for d in got] == list(range(gi.n))
    assert same(got[77].dist, O.gs_sssp(gi, 77)[0])
    assert agg is not None
    with pytest.raises(ValueError):
        P.mssp(gi, [0], schedule="chaotic")


def test_results_survive_later_calls_of_the_same_size(gpu):
    """Pooled page-locked result blocks: rows and slices of an
    earlier result must not be overwritten by a later call of the same size."""
    g = G.rmat_graph(10, 8, weights="int")
    a = P.mssp(g, [0, 1])
    a_rows = [dv.dist.copy() for dv, _ in a]
    view = a[0][0].dist[: g.n // 2]
    view_copy = view.copy()
    for srcs in ([2, 3], [4, 5], [6, 7], [8, 9], [10, 11]):
        P.mssp(g, srcs)
    d1 = P.govm_sssp(g, 5)[0].dist
    keep = d1[:10]
    P.mssp(g, [12])
    P.govm_sssp(g, 7)
    for (dv, _), ref in zip(a, a_rows):
        assert np.array_equal(dv.dist, ref)
    assert np.array_equal(view, view_copy)
    assert np.array_equal(keep, P.govm_sssp(g, 5)[0].dist[:10])
