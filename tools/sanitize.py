"""Small solves of every kernel family under compute-sanitizer (memcheck /
racecheck / synccheck): single-source GOVM/GSVM on all value types, frontier
modes and tile widths, both round schedules (async with the worklist tail off,
at the default and from round 2 on), predecessors + negative-cycle check,
batched multi-source (both schedules), device CSR build, device Floyd-Warshall,
the chunked host-graph upload.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np

import paper_2306_07872_b200 as P
from paper_2306_07872_b200 import devgen as D
from paper_2306_07872_b200 import generators as G
from paper_2306_07872_b200 import multisource as MS


def main():
    rng = np.random.default_rng(0)
    graphs = []
    for n, kind in ((300, "int"), (500, "float"), (5000, "grid"), (4096, "rmat")):
        if kind == "grid":
            graphs.append(G.grid_graph(70, 72))
        elif kind == "rmat":
            graphs.append(G.rmat_graph(12, 8, weights="f32"))
        else:
            m = 6 * n
            w = rng.integers(1, 30, m).astype(float) if kind == "int" else rng.uniform(0, 2, m)
            graphs.append(P.csr_from_arrays(n, rng.integers(0, n, m), rng.integers(0, n, m), w))
    neg, _ = G.johnson_reweight(G.rmat_graph(10, 8), pseed=3)
    cyc = G.inject_cycles(neg, 1, source=0, seed=7)
    checked = 0
    # round-1 kernel modes with the small-graph cluster kernel off, then the cluster kernel forced on
    for mode in ((0.5, -1, -1, 0), (1e9, 0, 1, 0), (0.0, 1, 0, 0), (1e9, 1, 0, 0), (0.5, -1, -1, 1)):
        P.set_tuning(dense_edges_per_node=mode[0], wide_tiles=mode[1], bitmap_frontier=mode[2], small_graph=mode[3])
        for g in graphs:
            for prec in ("auto", "fp32", "fp64"):
                for algo in ("govm", "gsvm"):
                    P.SOLVERS[algo](g, 0, precision=prec)
                    checked += 1
                for wl in (0.0, float(1 << 20), 1e18):  # async: tail off / default / from round 2
                    P.set_tuning(worklist_edges=wl)
                    P.govm_sssp(g, 0, precision=prec, schedule="async")
                    checked += 1
                P.set_tuning(worklist_edges=float(1 << 20))
            P.govm_sssp(g, 1, record_pred=True)
            MS.mssp_tile(g, list(range(40)), "govm")
            MS.mssp_tile(g, list(range(40)), "govm", schedule="async")
            MS.mssp_tile(g, list(range(7)), "gsvm")
            checked += 4
    P.set_tuning(dense_edges_per_node=0.5, wide_tiles=-1, bitmap_frontier=-1, small_graph=-1)
    for spec in (1, 0):  # negative weights: speculative plain kernel first / tracking kernel only
        P.set_tuning(speculate_negcheck=spec)
        for g in (neg, cyc):
            P.govm_sssp(g, 0)
            P.govm_sssp(g, 0, record_pred=True)
            P.gsvm_sssp(g, 0)
            checked += 3
    P.set_tuning(speculate_negcheck=1)
    # the near-far kernel (async, low degree): grid default, forced on an RMAT, tiny / huge buckets
    P.set_tuning(small_graph=0)
    for delta in (0.0, 1.0, 1e9):
        P.set_tuning(nearfar_delta=delta)
        P.govm_sssp(graphs[2], 0, schedule="async")
        checked += 1
    P.set_tuning(nearfar=1, nearfar_delta=0)
    P.govm_sssp(graphs[3], 0, precision="fp32", schedule="async")
    P.govm_sssp(graphs[0], 0, schedule="async")
    P.set_tuning(nearfar=-1, small_graph=-1)
    checked += 2
    # the priority window (async, persistent kernel): every round after the first dense one
    # histogrammed and windowed, on every graph and value type it applies to
    P.set_tuning(small_graph=0, dense_edges_per_node=0.0, priority_edges_per_edge=0.0)
    for frac in (0.35, 0.05):
        P.set_tuning(priority_frac=frac)
        for g in graphs:
            for prec in ("auto", "fp32"):
                P.govm_sssp(g, 0, precision=prec, schedule="async")
                checked += 1
    P.set_tuning(small_graph=-1, dense_edges_per_node=0.5, priority_edges_per_edge=0.4, priority_frac=0.2)
    u = rng.integers(0, 1000, 20000)
    v = rng.integers(0, 1000, 20000)
    D.build_csr_device(1000, u, v, rng.uniform(0, 1, 20000))
    P.floyd_warshall_apsp(graphs[0])
    P.floyd_warshall_apsp(neg if neg.n <= 2000 else graphs[1])
    big = G.rmat_graph(16, 80, weights="f32")  # m >= 2^22: chunked DMA upload path
    P.govm_sssp(big, 0, precision="fp32", schedule="async")
    print(f"sanitize: {checked} solves (persistent, priority window, worklist, near-far, small-graph cluster, speculative negative-weight) + batches + csr build + floyd-warshall + staged upload ran")


if __name__ == "__main__":
    main()
