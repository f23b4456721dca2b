"""Per-round device timeline of one C2-style solve (DAWN_F_PROFILE).

    python tools/round_profile.py [--scale 22] [--ef 16] [--weights f32] [--solves 3] [--algo govm]

Prints one row per round: frontier entries, frontier edges, S-phase and
X-phase durations (device globaltimer), and writes JSON to --out.  Also the
ncu target for the persistent kernel (short command line, few launches).
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--weights", default="f32")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--algo", default="govm")
    ap.add_argument("--source", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--grid", type=int, default=0, help="grid side (>0: 2D grid instead of RMAT)")
    ap.add_argument("--dense", type=float, default=None, help="dense_edges_per_node tuning knob")
    ap.add_argument("--bitmap", type=float, default=None, help="bitmap_edges_per_node tuning knob")
    ap.add_argument("--schedule", choices=["async", "jacobi"], default="async")
    ap.add_argument("--tune", action="append", default=[], help="key=value solver tuning (repeatable)")
    a = ap.parse_args()
    import torch

    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200.devgen import rmat_device_graph

    if a.grid:
        from paper_2306_07872_b200 import device as D
        from paper_2306_07872_b200 import generators as G

        g = G.grid_graph(a.grid, a.grid)
        dg = D.DeviceGraph.from_csr(g, precision="auto")
    else:
        dg, _, _ = rmat_device_graph(a.scale, a.ef, weights=a.weights, precision=a.precision)
    L = N.lib()
    s = dg.solver(N.F_PROFILE)
    if a.dense is not None:
        N.check(L.dawn_solver_tune(s, b"dense_edges_per_node", a.dense))
    for kv in a.tune:
        k_, v_ = kv.split("=")
        N.check(L.dawn_solver_tune(s, k_.encode(), float(v_)))
    if a.bitmap is not None:
        N.check(L.dawn_solver_tune(s, b"bitmap_edges_per_node", a.bitmap))
    stream = torch.cuda.current_stream().cuda_stream
    algo = N.GOVM if a.algo == "govm" else N.GSVM
    times = []
    for _ in range(a.solves):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(L.dawn_sssp_begin(s, a.source, algo, N.F_ASYNC if a.schedule == "async" else 0, stream))
        N.check(L.dawn_sssp_run(s, 0, stream))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    st = N.Stats()
    N.check(L.dawn_solver_result(s, None, None, ctypes.byref(st), stream))
    cap = 1 << 16
    buf = (ctypes.c_uint64 * (4 * cap))()
    nr = ctypes.c_int64(0)
    N.check(L.dawn_solver_round_profile(s, buf, cap, ctypes.byref(nr), stream))
    ebits = 64 - dg.n.bit_length()
    rows = []
    for r in range(1, nr.value):
        t0, t1, t2, pk = buf[4 * r], buf[4 * r + 1], buf[4 * r + 2], buf[4 * r + 3]
        if t0 == 0:
            continue
        rows.append({"round": r, "entries": pk >> ebits, "edges": pk & ((1 << ebits) - 1),
                     "s_us": (t1 - t0) / 1e3, "x_us": (t2 - t1) / 1e3})
    tot_s = sum(x["s_us"] for x in rows)
    tot_x = sum(x["x_us"] for x in rows)
    print(f"solve ms: {[round(t, 3) for t in times]}  rounds={st.outer_steps} R={st.relaxations} W={st.writes}")
    print(f"{'r':>4} {'entries':>10} {'edges':>12} {'S us':>8} {'X us':>9} {'Gedge/s':>8}")
    for x in rows:
        rate = x["edges"] / (x["x_us"] * 1e3) if x["x_us"] > 0 else 0
        print(f"{x['round']:>4} {x['entries']:>10} {x['edges']:>12} {x['s_us']:>8.1f} {x['x_us']:>9.1f} {rate:>8.1f}")
    print(f"sum S {tot_s:.1f} us, sum X {tot_x:.1f} us")
    wl = (ctypes.c_uint64 * 6)()
    N.check(L.dawn_solver_worklist_stats(s, wl, stream))
    if wl[1]:
        nwarps = max(1, (wl[3] + wl[4]) / max(wl[5], 1))
        print(f"worklist: from round {wl[0]}, {wl[1]} items in {wl[2]} warp batches "
              f"({wl[1] / max(wl[2], 1):.1f} items/batch), kernel span {wl[5] / 1e3:.1f} us, "
              f"busy {wl[3] / 1e3 / nwarps:.1f} us per warp of {nwarps:.0f}, "
              f"{wl[3] / max(wl[2], 1) / 1e3:.2f} us per batch")
    if rows and times:
        tail = min(times) * 1e3 - (buf[4 * rows[-1]["round"] + 2] - buf[4 * rows[0]["round"]]) / 1e3
        print(f"after the last recorded round (worklist kernel, if it ran, + launch gaps): {tail:.1f} us of the fastest solve")
    # per-CTA end of S / X work relative to the phase start (imbalance vs throughput)
    gridc = ctypes.c_int(0)
    cp = (ctypes.c_uint64 * (2 * 2048 * 64))()
    N.check(L.dawn_solver_cta_profile(s, cp, 64, ctypes.byref(gridc), stream))
    G = gridc.value
    print(f"{'r':>4} {'S min':>7} {'S med':>7} {'S max':>7} {'X min':>7} {'X med':>7} {'X max':>7}  (us after phase start, {G} CTAs)")
    import statistics as stt
    for x in rows:
        r = x["round"]
        if r >= 64:
            break
        t0, t1 = buf[4 * r], buf[4 * r + 1]
        se = [cp[(r * 2 + 0) * G + b] for b in range(G)]
        xe = [cp[(r * 2 + 1) * G + b] for b in range(G)]
        if min(se) == 0 or min(xe) == 0:
            continue
        fs = [(v - t0) / 1e3 for v in se]
        fx = [(v - t1) / 1e3 for v in xe]
        print(f"{r:>4} {min(fs):>7.1f} {stt.median(fs):>7.1f} {max(fs):>7.1f} {min(fx):>7.1f} {stt.median(fx):>7.1f} {max(fx):>7.1f}")
    if a.out:
        Path(a.out).write_text(json.dumps({"solve_ms": times, "rounds": rows, "R": st.relaxations,
                                           "W": st.writes, "steps": st.outer_steps}, indent=1))


if __name__ == "__main__":
    main()
