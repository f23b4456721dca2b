"""Golden outputs of the REFERENCE oracles (oracles.py: floyd_warshall_apsp,
bellman_ford_sssp, dijkstra_sssp) for the device oracles of
paper_2306_07872_b200.oracles.  Run in the build container
only (imports /root/reference/pkg/src):

    python tests/golden/make_oracle_golden.py

Writes tests/golden/oracles.npz (graphs + results) and oracles.json (index).
Cases: the reference tests' known-answer graphs (pkg/tests/conftest.py),
its random corpus (pkg/tests/_gen.py) in the uniform02 / mixed / unit regimes,
negative-cycle graphs, and a graph with parallel edges and self-loops.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import sparsepath as R  # noqa: E402
from _gen import graph_with_negative_cycle, random_graph  # noqa: E402


def make_csr(n, edges):
    return R.build_csr(R.EdgeList(n=n, edges=[(u, v, float(w)) for u, v, w in edges]))


def main() -> None:
    graphs = {
        "three_node": make_csr(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 3.0)]),
        "neg_cycle": make_csr(3, [(0, 1, 1.0), (1, 2, -5.0), (2, 1, 1.0)]),
        "hand_trace": make_csr(3, [(0, 1, 1.9), (0, 2, 0.1), (2, 1, 0.1)]),
        "neg_edge_path": make_csr(3, [(0, 1, 2.0), (0, 2, 5.0), (1, 2, -4.0)]),
        "unreachable_cycle": make_csr(4, [(0, 1, 1.0), (2, 3, -5.0), (3, 2, 1.0)]),
        "edgeless": make_csr(3, []),
        "parallel_self": make_csr(6, [(0, 1, 4.0), (0, 1, 2.5), (1, 1, 0.5), (1, 2, 1.0), (2, 0, 3.0),
                                      (2, 0, 7.0), (3, 4, 1.0), (4, 5, 0.25), (5, 3, 0.125), (0, 3, 10.0)]),
    }
    for seed in range(6):
        graphs[f"u02_{seed}"] = random_graph(seed, n=25, avg_degree=3.0, regime="uniform02")
        graphs[f"mix_{seed}"] = random_graph(seed, n=20, avg_degree=3.0, regime="mixed")
        graphs[f"unit_{seed}"] = random_graph(seed, n=60, avg_degree=4.0, regime="unit")
    for seed in range(3):
        graphs[f"ncy_{seed}"] = graph_with_negative_cycle(seed, n=30, avg_degree=3.0)[0]
    graphs["u02_big"] = random_graph(99, n=300, avg_degree=5.0, regime="uniform02")
    # zero weights, ties in the heap, duplicate (u, v) pairs with decreasing weights
    graphs["ties_zero"] = make_csr(6, [(0, 1, 0.0), (0, 2, 0.0), (1, 3, 1.0), (2, 3, 1.0), (3, 4, 0.0),
                                       (0, 4, 5.0), (0, 4, 3.0), (0, 4, 1.0), (4, 5, 0.5), (1, 5, 1.5)])
    graphs["ncy_source"] = make_csr(4, [(0, 1, 1.0), (1, 0, -3.0), (1, 2, 1.0), (2, 3, 1.0)])

    arrays: dict[str, np.ndarray] = {}
    index: dict[str, dict] = {}
    for name, g in graphs.items():
        arrays[f"{name}.row_ptr"] = np.asarray(g.row_ptr, dtype=np.int64)
        arrays[f"{name}.col"] = np.asarray(g.col, dtype=np.int64)
        arrays[f"{name}.val"] = np.asarray(g.val, dtype=np.float64)
        fw = R.floyd_warshall_apsp(g)
        arrays[f"{name}.fw"] = fw.matrix
        meta = {"n": g.n, "m": g.m, "fw_negative_cycle": fw.negative_cycle, "fw_relaxations": fw.relaxations,
                "sources": []}
        nonneg = g.m == 0 or float(np.min(g.val)) >= 0
        for s in sorted({0, g.n // 2, g.n - 1}):
            bf = R.bellman_ford_sssp(g, s)
            arrays[f"{name}.bf{s}"] = bf.dist.dist
            rec = {"source": s, "bf_negative_cycle": bf.negative_cycle, "bf_relaxations": bf.relaxations}
            if nonneg:
                dj = R.dijkstra_sssp(g, s)
                arrays[f"{name}.dj{s}"] = dj.dist.dist
                rec["dj_relaxations"] = dj.relaxations
            meta["sources"].append(rec)
        meta["nonneg"] = nonneg
        index[name] = meta
    np.savez_compressed(HERE / "oracles.npz", **arrays)
    (HERE / "oracles.json").write_text(json.dumps(index, indent=1))


if __name__ == "__main__":
    main()
