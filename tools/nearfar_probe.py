"""Bucket-width sweep of the near-far schedule (dawn_nearfar.cuh).

    python tools/nearfar_probe.py [--grid 4096] [--means 2,4,8,16,32] [--solves 3] [--rmat 0]

For each auto bucket width (nearfar_delta_mean x mean edge weight) times the
async solve through the C ABI (CUDA events, graph resident) and prints the
work counters; the distances are checked equal to the Jacobi solve.  With
--rmat S the graph is RMAT-S ef16 fp32 instead (near-far forced on).
"""
import argparse
import ctypes
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=4096)
    ap.add_argument("--rmat", type=int, default=0)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--weights", default="f32", help="rmat weights: f32 (fp32 U[0,1)) or int (1..100, exact path)")
    ap.add_argument("--means", default="2,4,8,16,32")
    ap.add_argument("--caps", default="8", help="nearfar_batches values (continuation batches per warp per round)")
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--source", type=int, default=0)
    ap.add_argument("--profile", default=None, help="MEAN,CAP: one profiled solve, per-round summary")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200 import device as D
    from paper_2306_07872_b200 import generators as G
    from paper_2306_07872_b200.devgen import rmat_device_graph

    if a.rmat:
        dg, _, _ = rmat_device_graph(a.rmat, a.ef, weights=a.weights,
                                     precision="fp32" if a.weights == "f32" else "auto")
        name = f"rmat{a.rmat}_ef{a.ef}_{a.weights}"
    else:
        dg = D.DeviceGraph.from_csr(G.grid_graph(a.grid, a.grid), precision="auto")
        name = f"grid{a.grid}"
    L = N.lib()
    s = dg.solver(0)
    stream = torch.cuda.current_stream().cuda_stream
    n = dg.n

    def solve(flags):
        ts = []
        for _ in range(a.solves):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(L.dawn_sssp_begin(s, a.source, N.GOVM, flags, stream))
            N.check(L.dawn_sssp_run(s, 0, stream))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        d = np.empty(n, np.float64)
        st = N.Stats()
        N.check(L.dawn_solver_result(s, d.ctypes.data, None, ctypes.byref(st), stream))
        return ts, d, st

    if a.profile:
        mean, cap = (float(x) for x in a.profile.split(","))
        sp = dg.solver(N.F_PROFILE)
        for k_, v_ in ((b"nearfar", 1.0), (b"nearfar_delta_mean", mean), (b"nearfar_batches", cap)):
            N.check(L.dawn_solver_tune(sp, k_, v_))
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(L.dawn_sssp_begin(sp, a.source, N.GOVM, N.F_ASYNC, stream))
            N.check(L.dawn_sssp_run(sp, 0, stream))
            e1.record()
            torch.cuda.synchronize()
        nr = ctypes.c_int64(0)
        buf = np.zeros((1 << 16, 4), dtype=np.uint64)
        N.check(L.dawn_solver_round_profile(sp, buf.ctypes.data, 1 << 16, ctypes.byref(nr), stream))
        k = int(nr.value)
        t = buf[1:k, 0].astype(np.int64)
        dt = np.diff(t) / 1e3
        nwarps = None
        print(f"profiled solve {e0.elapsed_time(e1):.3f} ms, rounds {k - 1}; us/round median {np.median(dt):.2f} "
              f"p90 {np.percentile(dt, 90):.2f} max {dt.max():.2f}")
        bs, bm, sw = buf[1:k, 1], buf[1:k, 2], buf[1:k, 3]
        print(f"batches/round mean {bs.mean():.0f}, max batches of one warp: median {np.median(bm):.0f} "
              f"p90 {np.percentile(bm, 90):.0f} max {bm.max()}; swept rows/round mean {sw.mean():.0f}")
        for i in list(range(1, min(k - 1, 8))) + list(range(k // 2, k // 2 + 5)):
            print(f"  r{i}: {dt[i - 1]:.1f} us, batches {bs[i - 1]}, max/warp {bm[i - 1]}, swept {sw[i - 1]}")
        return
    N.check(L.dawn_solver_tune(s, b"nearfar", 0.0))
    ts, dj, sj = solve(N.F_ASYNC)
    print(json.dumps({"graph": name, "mode": "async, near-far off", "ms": statistics.median(ts),
                      "relaxations": sj.relaxations, "writes": sj.writes, "rounds": sj.outer_steps}), flush=True)
    ts, dj, sj = solve(0)
    print(json.dumps({"graph": name, "mode": "jacobi", "ms": statistics.median(ts), "relaxations": sj.relaxations,
                      "writes": sj.writes, "rounds": sj.outer_steps}), flush=True)
    N.check(L.dawn_solver_tune(s, b"nearfar", 1.0))
    for mean, cap in [(float(x), float(c)) for x in a.means.split(",") for c in a.caps.split(",")]:
        N.check(L.dawn_solver_tune(s, b"nearfar_delta_mean", mean))
        N.check(L.dawn_solver_tune(s, b"nearfar_batches", cap))
        ts, d, st = solve(N.F_ASYNC)
        print(json.dumps({"graph": name, "mode": "near-far", "delta_mean": mean, "cap": cap, "ms": statistics.median(ts),
                          "ms_all": [round(x, 3) for x in ts], "relaxations": st.relaxations, "writes": st.writes,
                          "rounds": st.outer_steps, "fd_equal": st.first_discoveries == sj.first_discoveries,
                          "dist_equal": bool(np.array_equal(d, dj))}), flush=True)


if __name__ == "__main__":
    main()
