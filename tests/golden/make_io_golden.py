"""Golden behaviour of the REFERENCE graph loaders / writers (graph.py:145-386)
for paper_2306_07872_b200.graphio.  Run in the build container only (imports
/root/reference/pkg/src):

    python tests/golden/make_io_golden.py

Writes tests/golden/io_cases.json: for each input text the parsed EdgeList
(n, edges) or the raised exception (type, message); for a few graphs the
exact text the writers produce."""

from __future__ import annotations

import io
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import sparsepath as R  # noqa: E402

EDGE_LISTS = {
    "plain": "0 1 2.5\n1 2 0.5\n",
    "weightless": "0 1\n1 2\n2 0\n",
    "header": "5 2\n0 1 1.0\n3 4 2.0\n",
    "header_too_small": "2 2\n0 1\n3 4\n",
    "header_count_mismatch": "5 3\n0 1\n3 4\n",
    "comments": "% c\n# c\n\n0 1 3\n  1 0 4  \n",
    "bad_fields": "0 1 2 3\n",
    "bad_id": "0 x 1\n",
    "neg_id": "0 -1 1\n",
    "nonfinite": "0 1 inf\n",
    "nan": "0 1 nan\n",
    "bad_weight": "0 1 abc\n",
    "selfloop": "2 2 1.5\n0 2 1\n",
    "empty": "",
    "line3": "0 1\n1 2\n1 2 3 4\n",
}
MTX = {
    "general": "%%MatrixMarket matrix coordinate real general\n% c\n3 3 2\n1 2 0.5\n3 1 2\n",
    "pattern_sym": "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 3\n1 2\n2 2\n4 3\n",
    "rect": "%%MatrixMarket matrix coordinate real general\n2 5 1\n2 5 1.25\n",
    "no_banner": "3 3 1\n1 1 1\n",
    "array": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "bounds": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 1\n",
    "too_few": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "fields": "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1 5\n",
    "empty": "",
}


def outcome(fn):
    try:
        el = fn()
        return {"n": el.n, "edges": [[int(u), int(v), float(w)] for u, v, w in el.edges]}
    except Exception as e:  # noqa: BLE001
        return {"error": type(e).__name__, "message": str(e)}


def main() -> None:
    out = {"edgelist": {}, "edgelist_undirected": {}, "mtx": {}, "writers": {}}
    for k, txt in EDGE_LISTS.items():
        out["edgelist"][k] = {"text": txt, **outcome(lambda: R.load_edge_list(io.StringIO(txt)))}
        out["edgelist_undirected"][k] = outcome(lambda: R.load_edge_list(io.StringIO(txt), directed=False))
    for k, txt in MTX.items():
        out["mtx"][k] = {"text": txt, **outcome(lambda: R.load_matrix_market(io.StringIO(txt)))}
    graphs = {
        "small": R.build_csr(R.EdgeList(n=4, edges=[(0, 1, 0.1), (0, 1, 1 / 3), (2, 0, 1e300), (3, 3, 5e-324)])),
        "empty": R.build_csr(R.EdgeList(n=3, edges=[])),
    }
    for k, g in graphs.items():
        a, b = io.StringIO(), io.StringIO()
        R.write_edge_list(g, a)
        R.write_matrix_market(g, b)
        out["writers"][k] = {"n": g.n, "edges": [[int(u), int(v), float(w)] for u, v, w in R.to_edge_list(g).edges],
                             "edgelist": a.getvalue(), "mtx": b.getvalue()}
    (Path(__file__).with_name("io_cases.json")).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
