"""Full-scale golden records produced by running the REFERENCE itself.

Run in the build container only (it imports ``sparsepath`` from
/root/reference, which does not exist on the GPU box); takes ~4 minutes on 8
cores:

    python tests/golden/make_scale_golden.py

For each case the reference's ``govm_sssp`` (``solver.py:324-399``) is run on
the same ``CsrGraph`` arrays the GPU path solves, and the record keeps

* ``graph_sha256`` of the int64/int64/float64 CSR arrays (so a test can prove
  it rebuilt the identical graph),
* ``dist_sha256`` of the float64 distance vector (bit-exact pin),
* a seeded 4096-entry sample ``(index, value)`` of the distances (for the fp32
  path's 1e-6 relative check, which cannot use a hash),
* the reference's ``SolveStats`` and the reached count.

Cases:
  c2_src0        RMAT-22 ef16 float32-valued U[0,1), source 0   (config 2, ~2 min)
  c3_src{i}      RMAT-20 ef16 float32, sources from the config-3 sample
  c5a_src0       RMAT-18 ef16 Johnson-reweighted int (negative edges, no cycle)
  c5b12_reach    RMAT-12 ef8 int + 1 reachable injected negative cycle (flag)
  c5b12_unreach  same with an unreachable cycle (no flag)
  grid1024_src0  1024x1024 4-neighbour grid, int 1..100 (config 4's twin, ~3 min)
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from multiprocessing import Pool
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO))

OUT = HERE / "scale_golden.json"
SAMPLE = 4096


def graph_sha(row_ptr, col, val) -> str:
    h = hashlib.sha256()
    for a, dt in ((row_ptr, np.int64), (col, np.int64), (val, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def c3_sources(row_ptr, k: int = 8192) -> list[int]:
    """The config-3 source sample: default_rng(5) over out-degree >= 1, ascending (bench.py)."""
    cand = np.flatnonzero(np.diff(row_ptr) > 0)
    rng = np.random.default_rng(5)
    return sorted(int(x) for x in rng.choice(cand, size=min(k, cand.size), replace=False))


def build_case(name: str):
    """The graph of a case, built exactly as the GPU tests build it."""
    from oracle import oracle as O
    from paper_2306_07872_b200 import generators as G
    from paper_2306_07872_b200.graph import CsrGraph

    if name == "c2_src0":
        n, m, rp, col, val = O.rmat_csr(22, 16, weights="f32", seed=1, wseed=2)
        return CsrGraph(n=n, m=m, row_ptr=rp, col=col, val=val), [0]
    if name.startswith("c3_"):
        n, m, rp, col, val = O.rmat_csr(20, 16, weights="f32", seed=1, wseed=2)
        src = c3_sources(rp)
        return CsrGraph(n=n, m=m, row_ptr=rp, col=col, val=val), [src[0], src[len(src) // 2], src[-1]]
    if name == "c5a_src0":
        n, m, rp, col, val = O.rmat_csr(18, 16, weights="int", seed=1, wseed=2)
        g, _ = G.johnson_reweight(CsrGraph(n=n, m=m, row_ptr=rp, col=col, val=val), pseed=3)
        return g, [0]
    if name.startswith("c5b12_"):
        base = G.rmat_graph(12, 8, weights="int", seed=1, wseed=2)
        base, _ = G.johnson_reweight(base, pseed=3)
        return G.inject_cycles(base, 1, source=0, seed=4, reachable=name.endswith("_reach")), [0]
    if name == "grid1024_src0":
        return G.grid_graph(1024, 1024), [0]
    raise KeyError(name)


def run_case(name: str) -> dict:
    import sparsepath as R

    g, sources = build_case(name)
    rg = R.CsrGraph(n=g.n, m=g.m, row_ptr=g.row_ptr, col=g.col, val=g.val)
    rng = np.random.default_rng(7)
    idx = np.sort(rng.choice(g.n, size=min(SAMPLE, g.n), replace=False))
    out = {"n": int(g.n), "m": int(g.m), "graph_sha256": graph_sha(g.row_ptr, g.col, g.val), "runs": []}
    for s in sources:
        t0 = time.perf_counter()
        dv, _, st = R.govm_sssp(rg, int(s))
        dt = time.perf_counter() - t0
        d = np.asarray(dv.dist, dtype=np.float64)
        run = {"source": int(s), "stats": st.as_dict(), "seconds": dt,
               "dist_sha256": hashlib.sha256(d.tobytes()).hexdigest(),
               "reached": int(np.isfinite(d).sum()),
               "sample_idx": idx.tolist(), "sample_val": [float(x) for x in d[idx]]}
        if g.n <= 4096:
            run["dist"] = [float(x) for x in d]
        out["runs"].append(run)
        print(f"{name} source {s}: {dt:.1f} s, {st.outer_steps} steps, flag {st.negative_cycle}", flush=True)
    return out


CASES = ["c2_src0", "grid1024_src0", "c3_sample", "c5a_src0", "c5b12_reach", "c5b12_unreach"]


def main() -> None:
    names = sys.argv[1:] or CASES
    old = json.loads(OUT.read_text()) if OUT.exists() else {}
    with Pool(min(4, len(names))) as pool:
        for name, rec in zip(names, pool.map(run_case, names)):
            old[name] = rec
    OUT.write_text(json.dumps(old, indent=0, sort_keys=True))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
