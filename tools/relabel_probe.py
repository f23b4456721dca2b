"""Probe: does a degree-ordered vertex relabeling speed up the C2 solve?

Builds RMAT-22 on the device, relabels it on the host (in-degree descending),
uploads both graphs and times the same solve (source 0 -> its new id).
Distances must agree after the permutation.
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--solves", type=int, default=5)
    ap.add_argument("--order", default="indeg")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200.device import DeviceGraph
    from paper_2306_07872_b200.devgen import rmat_csr_device

    n, m, rp, col, val = rmat_csr_device(a.scale, 16, weights="f32")
    L = N.lib()
    stream = torch.cuda.current_stream().cuda_stream

    def solve(dg, src, hot=0):
        s = dg.solver(0)
        ts = []
        for _ in range(a.solves):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(L.dawn_sssp_begin(s, src, N.GOVM, 0, stream))
            N.check(L.dawn_sssp_run(s, 0, stream))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        d = torch.empty(dg.n, dtype=torch.float64, device="cuda")
        st = N.Stats()
        N.check(L.dawn_solver_result(s, d.data_ptr(), None, ctypes.byref(st), stream))
        return ts, d, st

    dg0 = DeviceGraph.from_device_arrays(n, m, rp, col, val, N.F32, 0)
    t0, d0, st0 = solve(dg0, 0)
    print(f"original : {[round(x, 3) for x in t0]}  R={st0.relaxations}")
    # relabel
    indeg = torch.bincount(col, minlength=n)
    outdeg = rp[1:] - rp[:-1]
    if a.order == "indeg":
        key = -indeg
    elif a.order == "both":
        key = -(indeg + outdeg)
    else:
        key = -outdeg
    order = torch.sort(key, stable=True).indices  # new -> old
    new_of_old = torch.empty_like(order)
    new_of_old[order] = torch.arange(n, device="cuda")
    u = torch.repeat_interleave(torch.arange(n, device="cuda"), outdeg)
    nu, nv = new_of_old[u], new_of_old[col]
    kk = nu * n + nv
    idx = torch.sort(kk, stable=True).indices
    ncol = nv[idx]
    nval = val[idx]
    cnt = torch.bincount(nu, minlength=n)
    nrp = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    torch.cumsum(cnt, 0, out=nrp[1:])
    del kk, idx, u, nu, nv
    dg1 = DeviceGraph.from_device_arrays(n, m, nrp, ncol, nval, N.F32, 0)
    s1 = int(new_of_old[0])
    t1, d1, st1 = solve(dg1, s1)
    print(f"relabeled: {[round(x, 3) for x in t1]}  R={st1.relaxations}  (source 0 -> {s1})")
    assert torch.equal(d1[new_of_old], d0), "distances differ after relabeling"
    assert st1.relaxations == st0.relaxations and st1.writes == st0.writes
    top = torch.sort(indeg, descending=True).values
    for f in (0.001, 0.01, 0.05):
        kf = int(n * f)
        print(f"top {f*100:.1f}% nodes ({kf}) receive {float(top[:kf].sum()) / m * 100:.1f}% of edges")
    print("distances and counters identical")


if __name__ == "__main__":
    main()
