"""Row output path (format_distance_row, solver.py:498-506):
the native formatter writes exactly the reference's text; the binary stream
round-trips.  Host-side code: runs in the CPU suite (the library loads
without a GPU)."""

from __future__ import annotations

import io
from math import inf

import numpy as np
import pytest

import paper_2306_07872_b200 as P


def ref_line(source, dist):  # the reference's expression, restated
    return ",".join([str(source)] + ["inf" if d == inf else "%.17g" % d for d in dist])


def sample_values(rng, n):
    v = np.concatenate([
        rng.uniform(0, 2, n // 4), rng.integers(0, 10**6, n // 8).astype(float), rng.standard_normal(n // 8) * 1e-300,
        rng.standard_normal(n // 8) * 1e300, rng.uniform(-5, 5, n // 8).astype(np.float32).astype(float),
        np.array([0.0, -0.0, inf, -inf, 5e-324, 1.7976931348623157e308, 0.1, 1 / 3, 100.0, 1e16, 1e17, 123456789012345678.0]),
    ])
    v = np.concatenate([v, np.full(n - v.size if n > v.size else 0, inf)])
    rng.shuffle(v)
    return v[:n]


@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (5000, 1), (300, 40), (0, 2)])
def test_native_text_equals_reference(n, k):
    rng = np.random.default_rng(n + k)
    rows = np.stack([sample_values(rng, n) for _ in range(k)]) if n else np.zeros((k, 0))
    src = [int(s) for s in rng.integers(0, 10**9, k)]
    got = P.format_distance_rows(rows, src)
    want = "".join(ref_line(s, r.tolist()) + "\n" for s, r in zip(src, rows))
    assert got == want


def test_format_distance_row_long_and_short_agree():
    rng = np.random.default_rng(3)
    d = sample_values(rng, 10000)
    dv = P.DistanceVector(dist=d, source=17)
    assert P.format_distance_row(dv) == ref_line(17, d.tolist())
    dv2 = P.DistanceVector(dist=d[:10], source=2)
    assert P.format_distance_row(dv2) == ref_line(2, d[:10].tolist())


def test_strided_rows_and_nan():
    big = np.full((3, 12), 7.25)
    big[1, 4] = np.nan
    rows = big[:, :9]
    txt = P.format_distance_rows(rows, [0, 1, 2])
    assert txt.splitlines()[1].split(",")[5] == "nan" and txt.count("\n") == 3


def test_binary_round_trip_and_errors():
    rng = np.random.default_rng(5)
    rows = rng.uniform(0, 1, (4, 33))
    rows[2, 7] = inf
    buf = io.BytesIO()
    nbytes = P.write_distance_rows(buf, rows, [9, 8, 7, 6], fmt="binary")
    assert nbytes == len(buf.getvalue()) == 8 + 16 + 4 * 8 + 4 * 33 * 8
    buf.seek(0)
    src, back = P.read_distance_rows(buf)
    assert src.tolist() == [9, 8, 7, 6] and np.array_equal(back, rows)
    t = io.BytesIO()
    P.write_distance_rows(t, rows, [9, 8, 7, 6])
    assert t.getvalue().decode() == P.format_distance_rows(rows, [9, 8, 7, 6])
    with pytest.raises(ValueError):
        P.write_distance_rows(t, rows, [1, 2, 3, 4], fmt="xml")
    with pytest.raises(ValueError):
        P.format_distance_rows(rows, [1, 2])


def test_random_bit_patterns_equal_python_formatting():
    rng = np.random.default_rng(11)
    v = rng.integers(0, 2**63, 50000, dtype=np.int64).view(np.float64)
    v = np.where(np.isnan(v), 1.5, v)
    assert P.format_distance_rows(v[None, :], [0]) == ref_line(0, v.tolist()) + "\n"
