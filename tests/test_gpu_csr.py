"""Device CSR construction (dawn_build_csr) against the
reference ordering of build_csr (graph.py:303-322): rows by source, columns
ascending, ties in input order, duplicates kept — bit-exact arrays."""

from __future__ import annotations

import numpy as np
import pytest
import torch
from conftest import make_csr

import paper_2306_07872_b200 as P
from paper_2306_07872_b200 import devgen as D
from paper_2306_07872_b200 import generators as G

pytestmark = pytest.mark.gpu


def same_graph(a, b) -> bool:
    return (a.n == b.n and a.m == b.m and np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col)
            and np.array_equal(a.val, b.val))


@pytest.mark.parametrize("seed", range(8))
def test_build_csr_matches_host_order(gpu, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(0, 20 * n))
    u = rng.integers(0, n, m)
    v = rng.integers(0, max(1, n // 7), m) if seed % 2 else rng.integers(0, n, m)  # many duplicates
    w = rng.uniform(-5, 5, m)
    host = P.csr_from_arrays(n, u, v, w)
    dev = D.build_csr_device(n, u, v, w)
    assert same_graph(dev, host)
    # device-resident inputs give the same arrays
    rp, col, val = D.csr_device(n, torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda(),
                                torch.from_numpy(w).cuda())
    assert np.array_equal(rp.cpu().numpy(), host.row_ptr) and np.array_equal(col.cpu().numpy(), host.col)
    assert np.array_equal(val.cpu().numpy(), host.val)


def test_build_csr_ties_keep_input_order(gpu):
    # parallel edges 0->1 with distinct weights must stay in input order (graph.py:318)
    el = P.EdgeList(n=3, edges=[(0, 1, 5.0), (2, 0, 1.0), (0, 1, 2.0), (0, 0, 7.0), (0, 1, 3.0)])
    host = P.build_csr(el)
    u, v, w = zip(*el.edges)
    dev = D.build_csr_device(3, np.array(u), np.array(v), np.array(w))
    assert same_graph(dev, host)
    assert dev.val.tolist() == [7.0, 5.0, 2.0, 3.0, 1.0]


def test_build_csr_edge_cases(gpu):
    e = D.build_csr_device(4, np.empty(0), np.empty(0), np.empty(0))
    assert e.m == 0 and e.row_ptr.tolist() == [0, 0, 0, 0, 0]
    with pytest.raises(ValueError, match="out of range"):
        D.build_csr_device(3, np.array([0, 3]), np.array([1, 1]), np.array([1.0, 1.0]))
    with pytest.raises(ValueError, match="non-finite"):
        D.build_csr_device(3, np.array([0]), np.array([1]), np.array([np.nan]))


def test_rmat_device_equals_host_generator(gpu):
    host = G.rmat_graph(14, 8, weights="int")  # config 1 built on the host
    n, m, rp, col, val = D.rmat_csr_device(14, 8, weights="int")
    dev = P.CsrGraph(n=n, m=m, row_ptr=rp.cpu().numpy(), col=col.cpu().numpy(), val=val.cpu().numpy())
    assert same_graph(dev, host)
    # and the solve on it matches
    a, _, sa = P.govm_sssp(host, 0)
    b, _, sb = P.govm_sssp(dev, 0)
    assert np.array_equal(a.dist, b.dist) and sa.as_dict() == sb.as_dict()


def test_build_csr_grid_scale(gpu):
    g = G.grid_graph(300, 300)
    u = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    perm = np.random.default_rng(3).permutation(g.m)
    dev = D.build_csr_device(g.n, u[perm], g.col[perm], g.val[perm])
    host = P.csr_from_arrays(g.n, u[perm], g.col[perm], g.val[perm])
    assert same_graph(dev, host)
    assert np.array_equal(dev.row_ptr, g.row_ptr)


@pytest.mark.parametrize("scale,ef,weights", [(14, 8, "int"), (18, 16, "f32"), (20, 16, "f32")])
def test_rmat_device_equals_reference_arm_generator(gpu, scale, ef, weights):
    """dawn_gen_rmat + dawn_build_csr (the bench's GPU arm) == the C generator
    the reference arm times (oracle rmat_csr): identical CsrGraph arrays."""
    from oracle import oracle as O

    n, m, rp, col, val = D.rmat_csr_device(scale, ef, weights=weights)
    on, om, orp, ocol, oval = O.rmat_csr(scale, ef, weights=weights)
    assert (n, m) == (on, om)
    assert np.array_equal(rp.cpu().numpy(), orp) and np.array_equal(col.cpu().numpy(), ocol)
    assert np.array_equal(val.cpu().numpy(), oval)


@pytest.mark.parametrize("rows,cols", [(1, 1), (1, 7), (9, 1), (2, 2), (3, 4), (57, 91), (300, 300), (1024, 1024)])
def test_grid_device_equals_host_generator(gpu, rows, cols):
    """dawn_gen_grid (closed-form CSR offsets, no sort) == generators.grid_graph."""
    host = G.grid_graph(rows, cols)
    n, m, rp, col, val = D.grid_csr_device(rows, cols)
    dev = P.CsrGraph(n=n, m=m, row_ptr=rp.cpu().numpy(), col=col.cpu().numpy(), val=val.cpu().numpy())
    assert same_graph(dev, host)


def test_grid_device_float_weights_and_solve(gpu):
    host = G.grid_graph(40, 50)
    n, m, rp, col, val = D.grid_csr_device(40, 50, weights="f32")
    assert np.array_equal(rp.cpu().numpy(), host.row_ptr) and np.array_equal(col.cpu().numpy(), host.col)
    assert np.array_equal(val.cpu().numpy(), G._weights(m, 2, "f32", 1, 100))
    dg, h2 = D.grid_device_graph(40, 50, precision="int32", keep_host=True)
    assert same_graph(h2, host) and (dg.n, dg.m) == (host.n, host.m)
    dg.close()


def test_grid_device_rejects_bad_shape(gpu):
    import ctypes

    from paper_2306_07872_b200 import _native as N

    assert N.lib().dawn_gen_grid(0, 0, 5, 0, 1, 100, 2, None, None, None, None) != 0
    assert N.lib().dawn_gen_grid(0, 3, 3, 0, 5, 1, 2, ctypes.c_void_p(8), ctypes.c_void_p(8), ctypes.c_void_p(8),
                                 None) != 0
