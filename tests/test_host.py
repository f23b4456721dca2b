"""Host-side logic that needs no GPU: argument checks in the reference's order,
containers, generators, stats arithmetic."""

from __future__ import annotations

from math import inf

import numpy as np
import pytest
from conftest import make_csr

import paper_2306_07872_b200 as P
from paper_2306_07872_b200 import generators as G


def test_source_checked_before_any_device_work(monkeypatch):
    g = make_csr(3, [(0, 1, 1.0)])
    # would raise RuntimeError if it got as far as the device
    with pytest.raises(ValueError, match="out of range"):
        P.govm_sssp(g, 3)
    with pytest.raises(ValueError, match="out of range"):
        P.gsvm_sssp(g, -1)
    with pytest.raises(ValueError, match="out of range"):
        P.mssp(g, [0, 7], "govm")
    with pytest.raises(ValueError, match="unknown solver"):
        P.mssp(g, [0], "dijkstra")
    with pytest.raises(ValueError, match="workers must be >= 1"):
        P.mssp(g, [0], "govm", workers=0)
    with pytest.raises(ValueError, match="unknown solver"):
        P.apsp(g, "bfs")


def test_no_cpu_fallback_without_gpu():
    from paper_2306_07872_b200 import _native as N

    if N.LIB_PATH.exists() and N.device_count() > 0:
        pytest.skip("a GPU is present")
    g = make_csr(3, [(0, 1, 1.0)])
    with pytest.raises(RuntimeError):
        P.govm_sssp(g, 0)


def test_csr_canonical_order_and_validation():
    g = make_csr(3, [(1, 2, 5.0), (0, 2, 1.0), (0, 1, 2.0), (0, 1, 0.5)])
    assert g.row_ptr.tolist() == [0, 3, 4, 4]
    assert g.col.tolist() == [1, 1, 2, 2]
    assert g.val.tolist() == [2.0, 0.5, 1.0, 5.0]  # ties keep input order
    assert not g.col.flags.writeable
    with pytest.raises(ValueError):
        P.CsrGraph(n=2, m=1, row_ptr=[0, 1, 0], col=[1], val=[1.0])
    with pytest.raises(ValueError):
        P.CsrGraph(n=2, m=1, row_ptr=[0, 1, 1], col=[5], val=[1.0])
    with pytest.raises(ValueError):
        P.CsrGraph(n=2, m=1, row_ptr=[0, 1, 1], col=[1], val=[np.inf])
    with pytest.raises(ValueError):
        P.build_csr(P.EdgeList(n=2, edges=[(0, 3, 1.0)]))
    rebuilt = P.build_csr(P.to_edge_list(g))
    assert rebuilt.col.tolist() == g.col.tolist() and rebuilt.val.tolist() == g.val.tolist()


def test_generate_random_graph_deterministic():
    a = P.generate_random_graph(50, 4.0, P.WeightMode.unit(), seed=3)
    b = P.generate_random_graph(50, 4.0, P.WeightMode.unit(), seed=3)
    assert a.col.tolist() == b.col.tolist()
    u = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    assert not np.any(u == a.col)  # no self loops
    w = P.apply_weight_mode(a, P.WeightMode.random_uniform(0, 2, 1))
    assert w.val.min() >= 0 and w.val.max() < 2


def test_grid_generator_shape():
    g = G.grid_graph(3, 4)
    assert g.n == 12 and g.m == 2 * (3 * 3 + 2 * 4)
    assert g.col[g.row_ptr[5]:g.row_ptr[6]].tolist() == [1, 4, 6, 9]
    assert g.val.min() >= 1 and g.val.max() <= 100


def test_rmat_generator_shape():
    g = G.rmat_graph(10, 8)
    assert g.n == 1024 and g.m == 8192
    assert g.out_degree(0) == max(g.out_degree(u) for u in range(g.n))  # vertex 0 is the hub


def test_johnson_has_negative_edges_no_cycles():
    base = G.rmat_graph(8, 4)
    g, p = G.johnson_reweight(base)
    assert g.val.min() < 0
    u = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    assert np.allclose(g.val - p[u] + p[g.col], base.val)


def test_stats_helpers():
    s1 = P.SolveStats(writes=3, first_discoveries=2, re_updates=1, mu=1.5, updated_ratio=0.5)
    s2 = P.SolveStats()
    agg = P.aggregate_stats([s1, s2])
    assert agg.sources == 2 and agg.reachable_sources == 1 and agg.mean_mu == 1.5
    d = s1.as_dict()
    assert set(map(type, d.values())) <= {int, float, bool}
    dv = P.DistanceVector(dist=np.array([0.0, 0.1, inf]), source=0)
    assert P.format_distance_row(dv) == "0,0,0.10000000000000001,inf"


def test_path_to():
    pv = P.PredecessorVector(pred=[None, 0, 1, None], source=0)
    assert pv.path_to(2) == [0, 1, 2]
    assert pv.path_to(0) == [0]
    assert pv.path_to(3) is None
    loop = P.PredecessorVector(pred=[None, 2, 1], source=0)
    assert loop.path_to(1) is None


def test_generate_random_graph_matches_reference_fixture():
    """The seeded ER generator reproduces the reference's graphs (graph.py:405-453)
    bit for bit: SHA-256 of row_ptr/col recorded from the reference."""
    import hashlib
    import json
    from pathlib import Path

    cases = json.loads((Path(__file__).resolve().parent / "golden" / "mu_reports.json").read_text())
    for c in cases:
        g = P.generate_random_graph(c["n"], c["avg_degree"], P.WeightMode.unit(), seed=c["graph_seed"])
        digest = hashlib.sha256(np.ascontiguousarray(g.row_ptr).tobytes() + np.ascontiguousarray(g.col).tobytes())
        assert digest.hexdigest() == c["graph_sha256"]


def test_pinned_result_pool_keeps_live_views(monkeypatch):
    """A pooled result block returns to the pool only when the last view of
    the result dies (row views of an mssp result kept the block's
    memory alive but not the array the finalizer watched)."""
    import gc

    import torch

    from paper_2306_07872_b200 import solver as S

    monkeypatch.setattr(S, "_new_pinned_block", lambda nbytes: torch.empty(nbytes, dtype=torch.uint8))
    monkeypatch.setattr(S, "_PINNED_FREE", {})
    monkeypatch.setattr(S, "_PINNED_LIVE", [0, 0])
    rows = S._host_array((2, 3))
    rows[:] = 1.0
    views = [rows[0], rows[1][1:]]
    del rows
    gc.collect()
    again = S._host_array((2, 3))  # must not reuse the block the views still point into
    again[:] = 2.0
    assert views[0].tolist() == [1.0, 1.0, 1.0] and views[1].tolist() == [1.0, 1.0]
    del views
    gc.collect()
    assert S._PINNED_FREE.get(48), "the block goes back to the pool once every view is gone"
    third = S._host_array(6)
    third[:] = 3.0
    assert again.tolist() == [[2.0] * 3] * 2


def test_mu_report_layout_matches_reference():
    """MuReport.to_dict / to_flat_dict keep the reference's key order
    (experiments.py:70-92)."""
    from paper_2306_07872_b200.experiments import MuReport

    a = P.AggregateStats(sources=2, writes=3).finish()
    b = P.AggregateStats(sources=2, writes=5).finish()
    r = MuReport("g", 2, a, b, 0.5, 1.25, 7, "n")
    d = r.to_dict()
    assert list(d) == ["graph_id", "sources_sampled", "baseline", "randomized", "mean_updated_ratio", "mean_mu",
                       "seed", "notes"]
    assert d["baseline"] == a.as_dict() and d["randomized"] == b.as_dict()
    f = r.to_flat_dict()
    keys = list(a.as_dict())
    assert list(f) == (["graph_id", "sources_sampled"] + [f"baseline_{k}" for k in keys]
                       + [f"randomized_{k}" for k in keys] + ["mean_updated_ratio", "mean_mu", "seed", "notes"])
    assert f["randomized_writes"] == 5 and f["baseline_writes"] == 3


def test_mu_experiment_validates_before_device_work():
    from paper_2306_07872_b200.experiments import run_mu_experiment

    g = P.generate_random_graph(10, 2.0, P.WeightMode.unit(), seed=1)
    with pytest.raises(ValueError, match="num_sources must be >= 1"):
        run_mu_experiment(g, num_sources=0)
    empty = P.generate_random_graph(0, 2.0, P.WeightMode.unit(), seed=1)
    with pytest.raises(ValueError, match="empty graph"):
        run_mu_experiment(empty, num_sources=3)
