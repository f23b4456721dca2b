"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports the reference package from
/root/reference, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz`` (arrays) and ``tests/golden/index.json``
(case metadata + the reference's SolveStats).  Cases:

* ``kat_*``   — the reference tests' known-answer graphs
                (pkg/tests/conftest.py:15-30, test_solver.py:32-129).
* ``rnd_*``   — the reference test corpus ``random_graph`` (pkg/tests/_gen.py:22-44)
                in all three weight regimes, solved by gsvm and govm.
* ``ncy_*``   — ``graph_with_negative_cycle`` (pkg/tests/_gen.py:47-69): flag cases.
* ``c1_*``    — BASELINE config 1 (RMAT-14, ef 8, int 1..100) from this package's
                counter-hash generator; graph stored as a SHA-256 of its arrays.
* ``f32_*``   — RMAT-12 ef16 with float32-valued weights (config 2 in miniature).
* ``jn_*``    — RMAT-10 with Johnson-potential negative weights (config 5a).
* ``grid_*``  — 24x24 grid, int weights (config 4 in miniature).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))
sys.path.insert(0, str(REPO))

import sparsepath as R  # noqa: E402
from sparsepath.solver import SOLVERS as REF_SOLVERS  # noqa: E402
from _gen import graph_with_negative_cycle, random_graph  # noqa: E402

from paper_2306_07872_b200 import generators as G  # noqa: E402


def graph_sha(g) -> str:
    h = hashlib.sha256()
    for a, dt in ((g.row_ptr, np.int64), (g.col, np.int64), (g.val, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    index: dict[str, dict] = {}

    def add(name, g, source, algo, store_graph=True, gen=None):
        rg = R.CsrGraph(n=g.n, m=g.m, row_ptr=g.row_ptr, col=g.col, val=g.val)
        dv, _, st = REF_SOLVERS[algo](rg, source)
        bf = R.bellman_ford_sssp(rg, source) if g.n <= 2000 else None
        arrays[f"{name}/dist"] = dv.dist
        if store_graph:
            arrays[f"{name}/row_ptr"] = np.asarray(g.row_ptr, np.int64)
            arrays[f"{name}/col"] = np.asarray(g.col, np.int64)
            arrays[f"{name}/val"] = np.asarray(g.val, np.float64)
        index[name] = {
            "n": int(g.n), "m": int(g.m), "source": int(source), "algo": algo,
            "stats": st.as_dict(), "graph_sha256": graph_sha(g), "stored_graph": store_graph,
            "generator": gen, "bf_negative_cycle": None if bf is None else bool(bf.negative_cycle),
        }

    def mk(n, edges):
        return R.build_csr(R.EdgeList(n=n, edges=[(u, v, float(w)) for u, v, w in edges]))

    kats = {
        "three_node": (mk(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 3.0)]), 0),
        "neg_cycle_graph": (mk(3, [(0, 1, 1.0), (1, 2, -5.0), (2, 1, 1.0)]), 0),
        "hand_trace": (mk(3, [(0, 1, 1.9), (0, 2, 0.1), (2, 1, 0.1)]), 0),
        "parallel_edges": (mk(2, [(0, 1, 2.0), (0, 1, 1.0)]), 0),
        "isolated_source": (mk(3, [(1, 2, 1.0)]), 0),
        "single_node": (mk(1, []), 0),
        "neg_self_loop": (mk(1, [(0, 0, -1.0)]), 0),
        "cycle_through_source": (mk(2, [(0, 1, 1.0), (1, 0, -5.0)]), 0),
        "unreachable_cycle": (mk(4, [(0, 1, 1.0), (2, 3, -5.0), (3, 2, 1.0)]), 0),
        "format_row": (mk(3, [(0, 1, 0.1)]), 0),
        "edgeless5": (mk(5, []), 3),
        "zero_weights": (mk(4, [(0, 1, 0.0), (1, 2, 0.0), (2, 1, 0.0), (2, 3, 2.5)]), 0),
    }
    for name, (g, s) in kats.items():
        for algo in ("govm", "gsvm"):
            add(f"kat_{name}_{algo}", g, s, algo)

    for regime in ("unit", "uniform02", "mixed"):
        for seed in range(12):
            g = random_graph(seed, n=25 + seed, avg_degree=3.0, regime=regime)
            for algo in ("govm", "gsvm"):
                add(f"rnd_{regime}_{seed}_{algo}", g, 0, algo)

    for seed in range(10):
        g, s = graph_with_negative_cycle(seed)
        for algo in ("govm", "gsvm"):
            add(f"ncy_{seed}_{algo}", g, s, algo)

    c1 = G.rmat_graph(14, 8, weights="int", lo=1, hi=100, seed=1, wseed=2)
    for s in (0, 1, 2, 3, 5, 8):
        add(f"c1_src{s}_govm", c1, s, "govm", store_graph=False,
            gen={"kind": "rmat", "scale": 14, "edge_factor": 8, "weights": "int", "lo": 1, "hi": 100, "seed": 1,
                 "wseed": 2})
    add("c1_src0_gsvm", c1, 0, "gsvm", store_graph=False,
        gen={"kind": "rmat", "scale": 14, "edge_factor": 8, "weights": "int", "lo": 1, "hi": 100, "seed": 1,
             "wseed": 2})

    f32 = G.rmat_graph(12, 16, weights="f32", seed=1, wseed=2)
    for s in (0, 7):
        add(f"f32_src{s}_govm", f32, s, "govm", store_graph=False,
            gen={"kind": "rmat", "scale": 12, "edge_factor": 16, "weights": "f32", "seed": 1, "wseed": 2})

    jn, _ = G.johnson_reweight(G.rmat_graph(10, 8, weights="int", lo=1, hi=100, seed=1, wseed=2), pseed=3)
    for s in (0, 4):
        add(f"jn_src{s}_govm", jn, s, "govm", store_graph=False,
            gen={"kind": "johnson_rmat", "scale": 10, "edge_factor": 8, "seed": 1, "wseed": 2, "pseed": 3})

    grid = G.grid_graph(24, 24)
    for algo in ("govm", "gsvm"):
        add(f"grid_src0_{algo}", grid, 0, algo, store_graph=False, gen={"kind": "grid", "rows": 24, "cols": 24})

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "index.json").write_text(json.dumps(index, indent=1, sort_keys=True))
    print(f"wrote {len(index)} cases")


if __name__ == "__main__":
    main()
