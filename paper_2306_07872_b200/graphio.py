"""Graph files, API-compatible with the reference's loaders and writers
(``graph.py:145-386`` of ``sparsepath``): whitespace edge lists with an
optional ``n m`` header, MatrixMarket coordinate (real / pattern, general /
symmetric), and ``read_graph`` / ``write_graph`` by extension.  Host-side
I/O (out of the device scope, kept as thin numpy for the
drop-in); the CSR they produce feeds the device path unchanged.

Semantics restated from the reference: comment lines start with ``%`` or
``#``; a missing weight is 1.0; weights must be finite; node ids are
non-negative integers; ``directed=False`` emits both directions (a self-loop
twice); the first two-token line is a header only when its ``m`` equals the
number of following edge lines and its ``n`` covers every id; MatrixMarket
indices are 1-based, ``n = max(rows, cols)``, symmetric off-diagonal entries
are mirrored, and the declared entry count must match.  Writers use ``%.17g``
(exact round trip) through the native formatter.
"""

from __future__ import annotations

import math
from pathlib import Path
from typing import IO, Iterable

import numpy as np

from .errors import GraphParseError, UnsupportedFormatError
from .graph import CsrGraph, EdgeList, build_csr

__all__ = ["load_edge_list", "load_matrix_market", "write_edge_list", "write_matrix_market", "read_graph",
           "write_graph"]


def _int_field(tok: str, line: int, what: str) -> int:
    try:
        x = int(tok)
    except ValueError:
        raise GraphParseError(f"expected integer {what}, got {tok!r}", line) from None
    if x < 0:
        raise GraphParseError(f"{what} must be non-negative, got {x}", line)
    return x


def _weight_field(tok: str, line: int) -> float:
    try:
        w = float(tok)
    except ValueError:
        raise GraphParseError(f"expected numeric weight, got {tok!r}", line) from None
    if not math.isfinite(w):
        raise GraphParseError(f"non-finite weight {tok!r} rejected", line)
    return w


def _content_lines(stream: Iterable[str], first_line: int = 1, comments: str = "%#"):
    for no, raw in enumerate(stream, start=first_line):
        t = raw.strip()
        if t and t[0] not in comments:
            yield no, t.split()


def load_edge_list(stream: Iterable[str], directed: bool = True) -> EdgeList:
    """``u v [w]`` lines (optionally headed by ``n m``) into an :class:`EdgeList`."""
    rows = []
    for no, tok in _content_lines(stream):
        if len(tok) not in (2, 3):
            raise GraphParseError(f"expected 'u v [w]', got {len(tok)} fields", no)
        rows.append((no, tok))
    header_n = None
    body = rows
    if rows and len(rows[0][1]) == 2:
        try:
            hn, hm = int(rows[0][1][0]), int(rows[0][1][1])
        except ValueError:
            hn, hm = -1, -1
        if hn >= 0 and hm == len(rows) - 1:
            top = -1
            ok = True
            for _, tok in rows[1:]:
                try:
                    top = max(top, int(tok[0]), int(tok[1]))
                except ValueError:
                    ok = False
                    break
            if ok and hn >= top + 1:
                header_n, body = hn, rows[1:]
    edges = []
    top = -1
    for no, tok in body:
        u = _int_field(tok[0], no, "node id")
        v = _int_field(tok[1], no, "node id")
        w = _weight_field(tok[2], no) if len(tok) == 3 else 1.0
        top = max(top, u, v)
        edges.append((u, v, w))
        if not directed:
            edges.append((v, u, w))
    return EdgeList(n=header_n if header_n is not None else top + 1, edges=edges)


def load_matrix_market(stream: Iterable[str]) -> EdgeList:
    """A MatrixMarket ``matrix coordinate`` stream into an :class:`EdgeList`."""
    it = iter(stream)
    banner = next(it, None)
    if banner is None:
        raise GraphParseError("empty stream, missing MatrixMarket banner", 1)
    parts = banner.strip().split()
    if len(parts) != 5 or parts[0].lower() != "%%matrixmarket":
        raise GraphParseError("missing '%%MatrixMarket' banner", 1)
    obj, fmt, field, sym = (x.lower() for x in parts[1:])
    if obj != "matrix" or fmt != "coordinate":
        raise UnsupportedFormatError(f"unsupported MatrixMarket variant '{obj} {fmt}': only 'matrix coordinate' "
                                     "is handled")
    if field not in ("real", "pattern"):
        raise UnsupportedFormatError(f"unsupported MatrixMarket field '{field}': only real/pattern are handled")
    if sym not in ("general", "symmetric"):
        raise UnsupportedFormatError(f"unsupported MatrixMarket symmetry '{sym}': only general/symmetric are "
                                     "handled")
    weighted = field == "real"
    nfields = 3 if weighted else 2
    shape = None
    edges = []
    count = 0
    for no, tok in _content_lines(it, first_line=2, comments="%"):
        if shape is None:
            if len(tok) != 3:
                raise GraphParseError("size line must be 'rows cols nnz'", no)
            shape = (_int_field(tok[0], no, "row count"), _int_field(tok[1], no, "column count"),
                     _int_field(tok[2], no, "entry count"))
            continue
        nr, nc, nnz = shape
        if len(tok) != nfields:
            raise GraphParseError(f"expected {nfields} fields per entry, got {len(tok)}", no)
        i = _int_field(tok[0], no, "row index")
        j = _int_field(tok[1], no, "column index")
        if not (1 <= i <= nr and 1 <= j <= nc):
            raise GraphParseError(f"entry ({i}, {j}) outside declared {nr} x {nc} bounds", no)
        w = _weight_field(tok[2], no) if weighted else 1.0
        count += 1
        if count > nnz:
            raise GraphParseError(f"more than the declared {nnz} entries", no)
        edges.append((i - 1, j - 1, w))
        if sym == "symmetric" and i != j:
            edges.append((j - 1, i - 1, w))
    if shape is None:
        raise GraphParseError("missing size line")
    if count != shape[2]:
        raise GraphParseError(f"declared {shape[2]} entries but found {count}")
    return EdgeList(n=max(shape[0], shape[1]), edges=edges)


def _edge_lines(g: CsrGraph, base: int) -> str:
    """``u v w`` lines in CSR order with ``%.17g`` weights (graph.py:339-356)."""
    if g.m == 0:
        return ""
    u = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(np.asarray(g.row_ptr, dtype=np.int64))) + base
    v = np.asarray(g.col, dtype=np.int64) + base
    return "".join("%d %d %.17g\n" % t for t in zip(u.tolist(), v.tolist(), np.asarray(g.val, dtype=np.float64).tolist()))


def write_edge_list(g: CsrGraph, fh: IO[str]) -> None:
    """``n m`` header, then one ``u v w`` line per edge (round-trips through :func:`load_edge_list`)."""
    fh.write(f"{g.n} {g.m}\n")
    fh.write(_edge_lines(g, 0))


def write_matrix_market(g: CsrGraph, fh: IO[str]) -> None:
    """``matrix coordinate real general`` with 1-based indices."""
    fh.write("%%MatrixMarket matrix coordinate real general\n")
    fh.write(f"{g.n} {g.n} {g.m}\n")
    fh.write(_edge_lines(g, 1))


def _fmt_of(path: Path) -> str:
    return "mtx" if path.suffix.lower() in (".mtx", ".mm") else "edgelist"


def read_graph(path, fmt: str | None = None, directed: bool = True) -> CsrGraph:
    """A graph file as CSR; the format follows the extension unless given."""
    path = Path(path)
    fmt = fmt or _fmt_of(path)
    if fmt not in ("mtx", "edgelist"):
        raise ValueError(f"unknown graph format {fmt!r}")
    with open(path, "r", encoding="utf-8") as fh:
        el = load_matrix_market(fh) if fmt == "mtx" else load_edge_list(fh, directed=directed)
    return build_csr(el)


def write_graph(g: CsrGraph, path, fmt: str | None = None) -> None:
    """Write a graph file; the format follows the extension unless given."""
    path = Path(path)
    fmt = fmt or _fmt_of(path)
    if fmt not in ("mtx", "edgelist"):
        raise ValueError(f"unknown graph format {fmt!r}")
    with open(path, "w", encoding="utf-8") as fh:
        (write_matrix_market if fmt == "mtx" else write_edge_list)(g, fh)
