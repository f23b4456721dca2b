"""Graph files (graph.py:145-386 of the reference): loaders and writers
against the reference's own outputs and errors (tests/golden/io_cases.json,
make_io_golden.py), plus round trips through read_graph / write_graph."""

from __future__ import annotations

import io
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2306_07872_b200 as P

CASES = json.loads((Path(__file__).parent / "golden" / "io_cases.json").read_text())


def outcome(fn):
    try:
        el = fn()
        return {"n": el.n, "edges": [[int(u), int(v), float(w)] for u, v, w in el.edges]}
    except Exception as e:  # noqa: BLE001
        return {"error": type(e).__name__, "message": str(e)}


def strip(d):
    return {k: v for k, v in d.items() if k != "text"}


@pytest.mark.parametrize("name", sorted(CASES["edgelist"]))
def test_edge_list_matches_reference(name):
    case = CASES["edgelist"][name]
    assert outcome(lambda: P.load_edge_list(io.StringIO(case["text"]))) == strip(case)
    assert outcome(lambda: P.load_edge_list(io.StringIO(case["text"]), directed=False)) == \
        CASES["edgelist_undirected"][name]


@pytest.mark.parametrize("name", sorted(CASES["mtx"]))
def test_matrix_market_matches_reference(name):
    case = CASES["mtx"][name]
    assert outcome(lambda: P.load_matrix_market(io.StringIO(case["text"]))) == strip(case)


@pytest.mark.parametrize("name", sorted(CASES["writers"]))
def test_writers_match_reference(name):
    case = CASES["writers"][name]
    g = P.build_csr(P.EdgeList(n=case["n"], edges=[tuple(e) for e in case["edges"]]))
    a, b = io.StringIO(), io.StringIO()
    P.write_edge_list(g, a)
    P.write_matrix_market(g, b)
    assert a.getvalue() == case["edgelist"]
    assert b.getvalue() == case["mtx"]


def test_read_write_graph_round_trip(tmp_path):
    rng = np.random.default_rng(2)
    n, m = 200, 1500
    g = P.csr_from_arrays(n, rng.integers(0, n, m), rng.integers(0, n, m), rng.uniform(0, 2, m))
    for ext in ("txt", "mtx", "mm", "el"):
        path = tmp_path / f"g.{ext}"
        P.write_graph(g, path)
        h = P.read_graph(path)
        assert h.n == g.n and np.array_equal(h.row_ptr, g.row_ptr) and np.array_equal(h.col, g.col)
        assert np.array_equal(h.val, g.val)  # %.17g round-trips exactly
    with pytest.raises(ValueError):
        P.write_graph(g, tmp_path / "x.txt", fmt="json")
    with pytest.raises(ValueError):
        P.read_graph(tmp_path / "g.txt", fmt="json")
    assert issubclass(P.GraphParseError, P.SparsepathError)
    e = P.GraphParseError("boom", 7)
    assert str(e) == "line 7: boom" and e.line == 7
