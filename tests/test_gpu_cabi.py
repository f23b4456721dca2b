"""The reference-facing C ABI exercised directly (the calls INTEGRATION.md
shows a maintainer adding): graph from the reference's host layout (pageable
and pinned), both schedules through dawn_sssp with host and device outputs,
dawn_mssp with host rows, repeated create/destroy (the memory pool), and the
worklist statistics — against the reference-generated golden fixtures."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch
from conftest import golden_dist, golden_graph, golden_index, golden_names

from paper_2306_07872_b200 import _native as N
from paper_2306_07872_b200 import generators as G

pytestmark = pytest.mark.gpu


def make(g, vtype, pinned=False):
    L = N.lib()
    rp, col, val = (np.ascontiguousarray(g.row_ptr, np.int64), np.ascontiguousarray(g.col, np.int64),
                    np.ascontiguousarray(g.val, np.float64))
    keep = (rp, col, val)
    if pinned:
        keep = tuple(torch.from_numpy(a.copy()).pin_memory() for a in (rp, col, val))
        ptrs = [t.data_ptr() for t in keep]
    else:
        ptrs = [a.ctypes.data for a in keep]
    h = C.c_void_p()
    N.check(L.dawn_graph_create(0, g.n, g.m, ptrs[0], ptrs[1] if g.m else None, ptrs[2] if g.m else None, vtype, 0,
                                C.byref(h)))
    return h, keep


@pytest.mark.parametrize("name", golden_names("rnd_")[:24] + golden_names("kat_"))
@pytest.mark.parametrize("flags", [0, N.F_ASYNC], ids=["jacobi", "async"])
def test_sssp_host_output(gpu, name, flags):
    meta = golden_index()[name]
    if meta["stats"]["negative_cycle"]:
        pytest.skip("distances are not defined under a negative cycle")
    g = golden_graph(name)
    L = N.lib()
    vt = C.c_int()
    N.check(L.dawn_choose_vtype(g.n, g.m, np.ascontiguousarray(g.val, np.float64).ctypes.data, 0, C.byref(vt)))
    h, keep = make(g, vt.value, pinned=bool(flags))
    s = C.c_void_p()
    N.check(L.dawn_solver_create(h, N.F_NEGCHECK, C.byref(s)))
    algo = N.GOVM if meta["algo"] == "govm" else N.GSVM
    out = np.empty(g.n)
    st = N.Stats()
    N.check(L.dawn_sssp(s, meta["source"], algo, N.F_NEGCHECK | flags, out.ctypes.data, None, C.byref(st), None))
    assert np.array_equal(out, golden_dist(name))
    assert st.first_discoveries == meta["stats"]["first_discoveries"]
    N.check(L.dawn_solver_destroy(s))
    N.check(L.dawn_graph_destroy(h))


def test_repeated_create_destroy_and_worklist_stats(gpu):
    L = N.lib()
    g = G.rmat_graph(16, 16, weights="f32")
    ref = None
    for it in range(6):
        h, keep = make(g, N.F32, pinned=it % 2 == 1)
        s = C.c_void_p()
        N.check(L.dawn_solver_create(h, 0, C.byref(s)))
        N.check(L.dawn_solver_tune(s, b"small_graph", 0.0))  # the worklist lives in the persistent kernels
        d = torch.empty(g.n, dtype=torch.float64, device="cuda")
        N.check(L.dawn_sssp(s, 0, N.GOVM, N.F_ASYNC, d.data_ptr(), None, None, None))
        wl = (C.c_uint64 * 6)()
        N.check(L.dawn_solver_worklist_stats(s, wl, None))
        assert wl[1] > 0 and wl[2] > 0 and wl[5] > 0  # the tail ran (2^20 default > this graph's rounds)
        h_out = d.cpu().numpy()
        if ref is None:
            ref = h_out
        assert np.array_equal(h_out, ref)
        N.check(L.dawn_sssp(s, 0, N.GOVM, 0, d.data_ptr(), None, None, None))
        assert np.array_equal(d.cpu().numpy(), ref)
        wl2 = (C.c_uint64 * 6)()
        N.check(L.dawn_solver_worklist_stats(s, wl2, None))
        assert wl2[1] == 0  # the Jacobi schedule never hands over
        N.check(L.dawn_solver_destroy(s))
        N.check(L.dawn_graph_destroy(h))


def test_mssp_host_rows_both_schedules(gpu):
    L = N.lib()
    g = golden_graph(golden_names("c1_")[0])
    h, keep = make(g, N.I32)
    s = C.c_void_p()
    N.check(L.dawn_solver_create(h, 0, C.byref(s)))
    src = np.arange(0, 40, dtype=np.int64)
    rows = {}
    for flags in (0, N.F_ASYNC):
        out = np.empty((src.size, g.n))
        sts = (N.Stats * src.size)()
        N.check(L.dawn_mssp(s, src.ctypes.data, src.size, N.GOVM, flags, out.ctypes.data, C.addressof(sts), None))
        rows[flags] = out
    assert np.array_equal(rows[0], rows[N.F_ASYNC])
    N.check(L.dawn_solver_destroy(s))
    N.check(L.dawn_graph_destroy(h))
