"""Small solves of every kernel family under compute-sanitizer (memcheck /
racecheck / synccheck): single-source GOVM/GSVM on all value types, frontier
modes and tile widths, predecessors + negative-cycle check, batched
multi-source, device CSR build.

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
    for mode in ((0.5, -1, -1), (1e9, 0, 1), (0.0, 1, 0), (1e9, 1, 0)):
        P.set_tuning(dense_edges_per_node=mode[0], wide_tiles=mode[1], bitmap_frontier=mode[2])
        for g in graphs:
            for prec in ("auto", "fp32", "fp64"):
                for algo in ("govm", "gsvm"):
                    P.SOLVERS[algo](g, 0, precision=prec)
                    checked += 1
            P.govm_sssp(g, 1, record_pred=True)
            MS.mssp_tile(g, list(range(40)), "govm")
            MS.mssp_tile(g, list(range(7)), "gsvm")
            checked += 3
    P.set_tuning(dense_edges_per_node=0.5, wide_tiles=-1, bitmap_frontier=-1)
    for g in (neg, cyc):
        P.govm_sssp(g, 0)
        P.govm_sssp(g, 0, record_pred=True)
        P.gsvm_sssp(g, 0)
        checked += 3
    u = rng.integers(0, 1000, 20000)
    v = rng.integers(0, 1000, 20000)
    D.build_csr_device(1000, u, v, rng.uniform(0, 1, 20000))
    print(f"sanitize: {checked} solves + batches + csr build ran")


if __name__ == "__main__":
    main()
