"""GPU parity: the CUDA path (through libdawn.so's C ABI) against the reference's
golden outputs and the oracle.  Bars: bit-exact distances for integer and
float64 weights, <= 1e-6 relative for the opt-in fp32 path, identical
negative-cycle flags, counters exactly equal to the snapshot-Jacobi oracle."""

from __future__ import annotations

import math
from math import inf

import numpy as np
import pytest
from conftest import golden_dist, golden_graph, golden_index, golden_names, is_integral, make_csr

import paper_2306_07872_b200 as P
from oracle import oracle as O
from paper_2306_07872_b200 import generators as G

pytestmark = pytest.mark.gpu

FP32_RTOL = 1e-6  # north_star tolerance for the fp32 path


def same(a, b) -> bool:
    return np.array_equal(np.asarray(a), np.asarray(b))


def counters(st: P.SolveStats) -> dict:
    return {"outer_steps": st.outer_steps, "relaxations": st.relaxations, "writes": st.writes,
            "first_discoveries": st.first_discoveries}


def oracle_counters(o: dict) -> dict:
    return {k: o[k] for k in ("outer_steps", "relaxations", "writes", "first_discoveries")}


def vt_name(g, precision):
    if precision == "fp32":
        return "float32"
    if precision == "fp64" or not is_integral(g):
        return "float64"
    return "int32"


# ---------------------------------------------------------------------------
# golden fixtures (reference outputs)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", golden_names())
def test_golden_cases(gpu, name):
    meta = golden_index()[name]
    g = golden_graph(name)
    solver = P.SOLVERS[meta["algo"]]
    for precision in ("auto", "fp64"):
        dv, _, st = solver(g, meta["source"], precision=precision)
        assert st.negative_cycle == meta["stats"]["negative_cycle"]
        if not meta["stats"]["negative_cycle"]:
            assert same(dv.dist, golden_dist(name)), precision
            assert st.first_discoveries == meta["stats"]["first_discoveries"]
        # counters equal the device-semantics oracle exactly
        _, _, o = O.jacobi_sssp(g, meta["source"], meta["algo"], vtype=vt_name(g, precision),
                                negcheck=vt_name(g, precision) == "int32")
        assert counters(st) == oracle_counters(o)
        assert st.updated_ratio == o["multi_written"] / max(o["first_discoveries"], 1)


@pytest.mark.parametrize("name", golden_names("f32_"))
def test_fp32_path(gpu, name):
    meta = golden_index()[name]
    g = golden_graph(name)
    dv, _, st = P.govm_sssp(g, meta["source"], precision="fp32")
    ref = golden_dist(name)
    fin = np.isfinite(ref)
    assert same(np.isfinite(dv.dist), fin)
    rel = np.abs(dv.dist[fin] - ref[fin]) / np.maximum(np.abs(ref[fin]), 1e-30)
    assert rel.max() <= FP32_RTOL
    od, _, o = O.jacobi_sssp(g, meta["source"], "govm", vtype="float32")
    assert same(dv.dist, od)  # same fp32 arithmetic, same fixpoint -> bit-exact vs oracle
    assert counters(st) == oracle_counters(o)


# ---------------------------------------------------------------------------
# reference test-suite behaviours (pkg/tests/test_solver.py), on the device
# ---------------------------------------------------------------------------
def test_seed_source(gpu, frontier_mode):
    g = make_csr(2, [(0, 1, 2.0), (0, 1, 1.0)])
    alpha, delta = [0.0, inf], [False, False]
    P.seed_source(g, 0, alpha, delta)
    assert alpha == [0.0, 1.0] and delta == [False, True]
    g = make_csr(3, [(1, 2, 1.0)])
    alpha, delta = [0.0, inf, inf], [False] * 3
    P.seed_source(g, 0, alpha, delta)
    assert alpha == [0.0, inf, inf] and delta == [False] * 3
    assert P.govm_sssp(g, 0)[2].outer_steps == 2
    g = make_csr(1, [(0, 0, -1.0)])
    st = P.SolveStats()
    alpha, delta = [0.0], [False]
    P.seed_source(g, 0, alpha, delta, stats=st)
    assert alpha == [0.0] and delta == [False] and st.writes == 0 and st.negative_cycle
    g = make_csr(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 3.0)])
    st = P.SolveStats()
    P.seed_source(g, 0, [0.0, inf, inf], [False] * 3, stats=st)
    assert st.first_discoveries == 2 and st.writes == 2 and st.relaxations == 2
    # duplicate source->j edges with decreasing weights: every improving edge
    # writes in CSR order, as in the reference (solver.py:231-249)
    g = make_csr(3, [(0, 1, 2.0), (0, 1, 1.0), (0, 1, 1.5), (0, 2, 0.5)])
    st, wc, pred = P.SolveStats(), [0, 0, 0], [None] * 3
    alpha, delta = P.seed_source(g, 0, [0.0, inf, inf], [False] * 3, stats=st, pred=pred, write_counts=wc)
    assert alpha == [0.0, 1.0, 0.5] and delta == [False, True, True]
    assert (st.writes, st.first_discoveries, st.relaxations) == (3, 2, 4)
    assert wc == [0, 2, 1] and pred == [None, 0, 0]


def test_hand_trace_and_small_cases(gpu):
    g = make_csr(3, [(0, 1, 1.9), (0, 2, 0.1), (2, 1, 0.1)])
    dv, _, st = P.govm_sssp(g, 0)
    assert dv.dist.tolist() == [0.0, 0.2, 0.1]
    assert (st.writes, st.first_discoveries, st.re_updates, st.mu, st.updated_ratio) == (3, 2, 1, 1.5, 0.5)
    g1 = make_csr(1, [])
    dv, _, st = P.gsvm_sssp(g1, 0)
    assert dv.dist.tolist() == [0.0] and st.outer_steps == 1 and st.writes == 0
    g2 = make_csr(2, [(0, 1, 1.0), (1, 0, -5.0)])
    dv, _, st = P.govm_sssp(g2, 0)
    assert st.negative_cycle and dv.dist[0] == 0.0
    g3 = make_csr(4, [(0, 1, 1.0), (2, 3, -5.0), (3, 2, 1.0)])
    assert not P.govm_sssp(g3, 0)[2].negative_cycle


def test_unit_weights_mu_one(gpu):
    g = P.generate_random_graph(200, 6.0, P.WeightMode.unit(), seed=11)
    _, _, st = P.govm_sssp(g, 0)
    assert st.re_updates == 0 and st.mu == 1.0
    agg = P.apsp(P.generate_random_graph(60, 4.0, P.WeightMode.unit(), seed=9), "govm")
    assert agg.re_updates == 0 and agg.mean_mu == 1.0


def test_predecessors(gpu):
    g = make_csr(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 3.0)])
    _, pv, _ = P.govm_sssp(g, 0, record_pred=True)
    assert pv.pred[0] is None and pv.path_to(2) == [0, 1, 2] and pv.path_to(0) == [0]
    _, pv, _ = P.govm_sssp(make_csr(3, [(1, 2, 1.0)]), 0, record_pred=True)
    assert pv.path_to(1) is None
    for name in golden_names("rnd_mixed_"):
        g = golden_graph(name)
        for solver in (P.govm_sssp, P.gsvm_sssp):
            dv, pv, st = solver(g, 0, record_pred=True)
            _, opred, _ = O.jacobi_sssp(g, 0, "govm" if solver is P.govm_sssp else "gsvm", vtype="float64",
                                        record_pred=True)
            assert [(-1 if p is None else p) for p in pv.pred] == opred.tolist()
            min_w = {}
            for u in range(g.n):
                for k in range(g.row_ptr[u], g.row_ptr[u + 1]):
                    key = (u, int(g.col[k]))
                    min_w[key] = min(float(g.val[k]), min_w.get(key, inf))
            for j in range(g.n):
                if dv.dist[j] == inf or j == 0:
                    continue
                path = pv.path_to(j)
                assert path is not None and path[0] == 0 and path[-1] == j
                total = sum(min_w[(a, b)] for a, b in zip(path, path[1:]))
                assert math.isclose(total, dv.dist[j], rel_tol=0.0, abs_tol=1e-9)


def test_trace_frontier_soundness(gpu, frontier_mode):
    for name in golden_names("rnd_uniform02_")[:8]:
        g = golden_graph(name)
        records = []
        dv, _, st = P.govm_sssp(g, 0, trace=lambda *a: records.append(a))
        dv2, _, st2 = P.govm_sssp(g, 0)
        assert same(dv.dist, dv2.dist) and st.as_dict() == st2.as_dict()
        assert len(records) == st.outer_steps - 1
        prev_w = prev_a = None
        for step, scanned, written, alpha in records:
            assert scanned == sorted(scanned) and written == sorted(written)
            if prev_w is not None:
                assert scanned == prev_w
            if prev_a is not None:
                assert all(a <= b for a, b in zip(alpha, prev_a))
            prev_w, prev_a = written, alpha
        if records:
            nbrs = {int(c) for c in g.col[g.row_ptr[0]:g.row_ptr[1]]}
            assert set(records[0][1]) <= nbrs
        assert sum(len(r[2]) for r in records) + len(records[0][1] if records else []) == st.writes


def test_mssp_apsp(gpu):
    g = golden_graph("rnd_uniform02_5_govm")
    rows = P.mssp(g, range(g.n), "govm")
    for s, (dv, st) in enumerate(rows):
        dv1, _, st1 = P.govm_sssp(g, s)
        assert dv.source == s and same(dv.dist, dv1.dist) and st.as_dict() == st1.as_dict()
    par = P.mssp(g, range(g.n), "govm", workers=4)
    assert all(same(a[0].dist, b[0].dist) and a[1].as_dict() == b[1].as_dict() for a, b in zip(rows, par))
    got = []
    agg = P.apsp(g, "gsvm", sink=got.append)
    assert [dv.source for dv in got] == list(range(g.n))
    assert all(same(a.dist, b[0].dist) for a, b in zip(got, rows))
    ref = P.aggregate_stats(P.gsvm_sssp(g, s)[2] for s in range(g.n))
    assert agg.as_dict() == ref.as_dict()
    e = make_csr(5, [])
    got = []
    agg = P.apsp(e, "govm", sink=got.append)
    assert len(got) == 5 and agg.reachable_sources == 0
    for dv in got:
        want = [inf] * 5
        want[dv.source] = 0.0
        assert dv.dist.tolist() == want

    def bad(dv):
        raise RuntimeError("boom")

    with pytest.raises(RuntimeError, match="boom"):
        P.apsp(e, "govm", sink=bad)


def test_determinism_and_stream_reuse(gpu):
    g = G.rmat_graph(14, 8)
    a = P.govm_sssp(g, 0)
    for _ in range(3):
        b = P.govm_sssp(g, 0)
        assert same(a[0].dist, b[0].dist) and a[2].as_dict() == b[2].as_dict()


# ---------------------------------------------------------------------------
# randomized parity against the oracle, all value types
# ---------------------------------------------------------------------------
@pytest.fixture(params=[(0.5, -1, -1, -1), (0.0, 1, 0, 0), (1e9, 1, 0, 0), (0.0, 0, 0, 0), (1e9, 0, 1, 0),
                        (0.5, 0, 1, 0), (0.5, -1, -1, 1)],
                ids=["auto", "all-dense-wide", "all-sparse-wide", "all-dense-narrow", "all-bitmap", "mixed-bitmap",
                     "small-cta"])
def frontier_mode(request):
    """Run under the default policy and the extremes of the persistent kernel
    (the one-CTA small-graph kernel off): stamps (dense) vs enqueue (sparse) vs
    bitmap light-round frontiers, 14- vs 8-edge-per-lane tiles; and the
    small-graph kernel forced on wherever it fits."""
    dense, wide, fb, small = request.param
    P.set_tuning(dense_edges_per_node=dense, wide_tiles=wide, bitmap_frontier=fb, small_graph=small)
    yield request.param
    P.set_tuning(dense_edges_per_node=0.5, wide_tiles=-1, bitmap_frontier=-1, small_graph=-1)


@pytest.mark.parametrize("seed", range(24))
def test_random_graphs_vs_oracle(gpu, seed, frontier_mode):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 400))
    m = int(rng.integers(0, 6 * n))
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    kind = seed % 4
    if kind == 0:
        w = rng.integers(1, 50, m).astype(float)
    elif kind == 1:
        w = rng.uniform(0, 2, m)
    elif kind == 2:  # negative weights on a DAG (no cycles)
        lo, hi = np.minimum(u, v), np.maximum(u, v)
        keep = lo != hi
        u, v = lo[keep], hi[keep]
        w = rng.integers(-20, 30, u.size).astype(float)
    else:
        w = rng.uniform(0, 1, m).astype(np.float32).astype(float)
    g = P.csr_from_arrays(n, u, v, w)
    src = int(rng.integers(0, n))
    for algo in ("govm", "gsvm"):
        for precision in ("auto", "fp64", "fp32"):
            vt = vt_name(g, precision)
            dv, _, st = P.SOLVERS[algo](g, src, precision=precision)
            od, _, o = O.jacobi_sssp(g, src, algo, vtype=vt, negcheck=vt == "int32")
            assert same(dv.dist, od), (algo, precision)
            assert counters(st) == oracle_counters(o)
            assert bool(st.negative_cycle) == bool(o["negative_cycle"])
        gd, _, gst = O.gs_sssp(g, src, algo)
        if not gst["negative_cycle"]:
            assert same(P.SOLVERS[algo](g, src)[0].dist, gd)  # vs the reference-order port


# ---------------------------------------------------------------------------
# negative cycles (config 5 in miniature and at scale)
# ---------------------------------------------------------------------------
def test_negative_cycles_rmat(gpu, frontier_mode):
    base, _ = G.johnson_reweight(G.rmat_graph(12, 16), pseed=3)
    dv, _, st = P.govm_sssp(base, 0)
    od, _, o = O.jacobi_sssp(base, 0, "govm", vtype="int32")
    assert not st.negative_cycle and same(dv.dist, od)
    gd, _, _ = O.gs_sssp(base, 0)
    assert same(dv.dist, gd)
    for k, reach in ((1, True), (4, True), (1, False)):
        cg = G.inject_cycles(base, k, source=0, seed=7, reachable=reach)
        _, _, st = P.govm_sssp(cg, 0)
        _, _, o = O.jacobi_sssp(cg, 0, "govm", vtype="int32", negcheck=True)
        assert st.negative_cycle == reach == bool(o["negative_cycle"])
        assert counters(st) == oracle_counters(o)
        _, _, stg = P.gsvm_sssp(cg, 0)
        assert stg.negative_cycle == reach


def test_negative_cycle_cap_without_early_exit(gpu):
    """Float weights take the reference's n-round cap path."""
    for seed in range(6):
        g, s = _ref_like_negative_cycle(seed)
        _, _, st = P.govm_sssp(g, s)
        _, _, o = O.jacobi_sssp(g, s, "govm", vtype="float64")
        assert st.negative_cycle and o["negative_cycle"] and st.outer_steps == g.n == o["outer_steps"]
        assert counters(st) == oracle_counters(o)


def _ref_like_negative_cycle(seed, n=40):
    rng = np.random.default_rng(seed)
    m = 4 * n
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    w = rng.uniform(0, 2, m)
    cyc = 1 + rng.choice(n - 1, size=3, replace=False)  # avoid the source: the cap path, not the guard
    eu = [cyc[0], cyc[1], cyc[2], 0]
    ev = [cyc[1], cyc[2], cyc[0], cyc[0]]
    ew = [0.5, 0.5, -1.5, 1.0]
    return P.csr_from_arrays(n, np.r_[u, eu], np.r_[v, ev], np.r_[w, ew]), 0


# ---------------------------------------------------------------------------
# larger graphs: exact vs oracle, properties at full scale
# ---------------------------------------------------------------------------
def test_rmat16_vs_oracle(gpu, frontier_mode):
    g = G.rmat_graph(16, 16, weights="f32")
    for precision, vt in (("fp32", "float32"), ("fp64", "float64")):
        dv, _, st = P.govm_sssp(g, 0, precision=precision)
        od, _, o = O.jacobi_sssp(g, 0, "govm", vtype=vt)
        assert same(dv.dist, od) and counters(st) == oracle_counters(o)
    gi = G.rmat_graph(16, 16, weights="int")
    dv, _, st = P.govm_sssp(gi, 0)
    gd, _, _ = O.gs_sssp(gi, 0)
    assert same(dv.dist, gd)


def test_grid_vs_oracle(gpu, frontier_mode):
    g = G.grid_graph(128, 128)
    for algo in ("govm", "gsvm"):
        dv, _, st = P.SOLVERS[algo](g, 0)
        od, _, o = O.jacobi_sssp(g, 0, algo, vtype="int32")
        assert same(dv.dist, od) and counters(st) == oracle_counters(o)
    gd, _, _ = O.gs_sssp(g, 0)
    assert same(dv.dist, gd)


def test_fixpoint_property_full_scale(gpu):
    """At BASELINE scale (RMAT-20 here; bench covers RMAT-22): the result is a
    fixpoint of the relax operator, the source is pinned, and the reached set
    is exactly the BFS-reachable set — size-independent checks."""
    import torch

    g = G.rmat_graph(20, 16, weights="f32")
    dv, _, st = P.govm_sssp(g, 0, precision="fp32")
    d = torch.from_numpy(dv.dist.astype(np.float32)).cuda()
    rp = torch.from_numpy(g.row_ptr).cuda()
    u = torch.repeat_interleave(torch.arange(g.n, device="cuda"), rp[1:] - rp[:-1])
    v = torch.from_numpy(g.col).cuda()
    w = torch.from_numpy(g.val.astype(np.float32)).cuda()
    cand = d[u] + w
    fin = torch.isfinite(d[u])
    assert bool(((d[v] <= cand) | ~fin | (v == 0)).all())
    assert dv.dist[0] == 0.0
    reach = torch.zeros(g.n, dtype=torch.bool, device="cuda")
    reach[0] = True
    while True:
        nxt = reach.clone()
        nxt[v[reach[u]]] = True
        if bool((nxt == reach).all()):
            break
        reach = nxt
    assert same(reach.cpu().numpy(), np.isfinite(dv.dist))
    assert st.first_discoveries == int(reach.sum()) - 1
