"""Breakdown of the end-to-end C-ABI step of bench.py (config 2): graph upload
from the reference's host layout, solver creation, solve with host output,
teardown — and the plain pinned H2D copy bandwidth for comparison.

    python tools/e2e_probe.py [--scale 22] [--steps 5]
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200 import generators as G

    g = G.rmat_graph(a.scale, 16, weights="f32")
    n, m = g.n, g.m
    rp = torch.from_numpy(np.array(g.row_ptr)).pin_memory()
    col = torch.from_numpy(np.array(g.col)).pin_memory()
    val = torch.from_numpy(np.array(g.val)).pin_memory()
    out = torch.empty(n, dtype=torch.float64).pin_memory()
    L = N.lib()
    stream = torch.cuda.current_stream().cuda_stream
    st = N.Stats()

    def timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return r, (time.perf_counter() - t0) * 1e3

    parts = {"graph_create": [], "solver_create": [], "sssp": [], "solver_destroy": [], "graph_destroy": []}
    for it in range(a.steps + 1):
        h = C.c_void_p()
        _, t = timed(lambda: N.check(L.dawn_graph_create(0, n, m, rp.data_ptr(), col.data_ptr(), val.data_ptr(),
                                                         N.F32, 0, C.byref(h))))
        parts["graph_create"].append(t)
        sv = C.c_void_p()
        _, t = timed(lambda: N.check(L.dawn_solver_create(h, 0, C.byref(sv))))
        parts["solver_create"].append(t)
        _, t = timed(lambda: N.check(L.dawn_sssp(sv, 0, N.GOVM, N.F_ASYNC, out.data_ptr(), None, C.byref(st),
                                                 stream)))
        parts["sssp"].append(t)
        _, t = timed(lambda: N.check(L.dawn_solver_destroy(sv)))
        parts["solver_destroy"].append(t)
        _, t = timed(lambda: N.check(L.dawn_graph_destroy(h)))
        parts["graph_destroy"].append(t)
    for k, v in parts.items():
        print(f"{k:>15}: {np.median(v[1:]):8.2f} ms  (first {v[0]:.2f})")
    byts = rp.numel() * 8 + col.numel() * 8 + val.numel() * 8
    d = [torch.empty(x.numel(), dtype=x.dtype, device="cuda") for x in (rp, col, val)]
    ts = []
    for _ in range(a.steps):
        _, t = timed(lambda: [y.copy_(x, non_blocking=True) for x, y in zip((rp, col, val), d)])
        ts.append(t)
    print(f"pinned H2D copy of the same {byts / 1e9:.3f} GB: {np.median(ts):.2f} ms = {byts / np.median(ts) / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
