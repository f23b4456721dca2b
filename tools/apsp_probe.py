"""Single-GPU timing probe of the batched multi-source kernel on config 3
(RMAT-20 ef16 float32 weights) — the per-batch cost and the single-source
loop it replaces.

    python tools/apsp_probe.py [--scale 20] [--k 1024] [--single 32]
"""
import argparse
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--k", type=int, default=1024)
    ap.add_argument("--single", type=int, default=32)
    ap.add_argument("--algo", default="govm")
    ap.add_argument("--order", default="id", help="batch grouping of the sources: id | degree | random")
    ap.add_argument("--util", type=float, default=None, help="batch_sparse_util tuning knob")
    ap.add_argument("--schedule", choices=["jacobi", "async"], default="async")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200 import multisource as MS
    from paper_2306_07872_b200.devgen import rmat_device_graph

    dg, _, deg = rmat_device_graph(a.scale, a.ef, weights="f32", precision="fp32")
    degh = deg.cpu().numpy()
    rng = np.random.default_rng(5)
    src = sorted(int(x) for x in rng.choice(np.flatnonzero(degh > 0), size=a.k, replace=False))
    if a.order == "degree":
        src = sorted(src, key=lambda x: (-int(degh[x]), x))
    elif a.order == "random":
        src = [src[i] for i in np.random.default_rng(9).permutation(len(src))]
    if a.util is not None:
        for fl in (0, N.F_PROFILE):
            N.check(N.lib().dawn_solver_tune(dg.solver(fl), b"batch_sparse_util", a.util))
    tile = torch.empty((a.k, dg.n), dtype=torch.float32, device="cuda")
    MS.mssp_tile(dg, src[:64], a.algo, out=tile[:64], stats=True, schedule=a.schedule)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, stats = MS.mssp_tile(dg, src, a.algo, out=tile, stats=True, schedule=a.schedule)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    R = sum(s.relaxations for s in stats)
    print(f"batched: k={a.k} {ms:.1f} ms  {a.k / ms * 1e3:.0f} sources/s  R={R:.3e} {R / ms / 1e6:.1f} G relax/s "
          f"per-batch {ms / ((a.k + 31) // 32):.3f} ms  mean steps {np.mean([s.outer_steps for s in stats]):.1f}")
    # single-source loop on the same sources
    L = N.lib()
    s = dg.solver(0)
    stream = torch.cuda.current_stream().cuda_stream
    ks = min(a.single, a.k)
    st = N.Stats()
    e0.record()
    for i in range(ks):
        N.check(L.dawn_sssp_begin(s, src[i], N.GOVM, 0, stream))
        N.check(L.dawn_sssp_run(s, 0, stream))
    e1.record()
    torch.cuda.synchronize()
    ms1 = e0.elapsed_time(e1)
    print(f"single loop: k={ks} {ms1:.1f} ms  {ks / ms1 * 1e3:.0f} sources/s")
    # cross-check a few rows against single solves
    for i in (0, ks // 2, ks - 1):
        N.check(L.dawn_sssp(s, src[i], N.GOVM if a.algo == "govm" else N.GSVM, 0, None, None, ctypes.byref(st),
                            stream))
        d = torch.empty(dg.n, dtype=torch.float64, device="cuda")
        N.check(L.dawn_solver_result(s, d.data_ptr(), None, ctypes.byref(st), stream))
        assert torch.equal(d, tile[i].double()), i
        if a.schedule == "jacobi":  # async counters are timing-dependent
            assert st.relaxations == stats[i].relaxations and st.writes == stats[i].writes, i
    print("rows match single-source solves")
    # per-round timeline of one batch (DAWN_F_PROFILE solver)
    sp = dg.solver(N.F_PROFILE)
    arr = np.ascontiguousarray(src[:32], dtype=np.int64)
    st32 = (N.Stats * 32)()
    N.check(L.dawn_mssp_batch(sp, arr.ctypes.data, 32, N.GOVM if a.algo == "govm" else N.GSVM,
                              N.F_ASYNC if a.schedule == "async" else 0, None, N.F64,
                              dg.n, ctypes.addressof(st32), stream))
    cap = 256
    buf = (ctypes.c_uint64 * (4 * cap))()
    nr = ctypes.c_int64(0)
    N.check(L.dawn_solver_round_profile(sp, buf, cap, ctypes.byref(nr), stream))
    ebits = 64 - dg.n.bit_length()
    print(f"{'r':>3} {'entries':>9} {'edges':>11} {'lane-edges':>12} {'util':>5} {'B us':>7} {'X us':>8} {'Gstep/s':>8}")
    tb = tx = 0.0
    for r in range(1, nr.value):
        t0, t1, pk, le = buf[4 * r], buf[4 * r + 1], buf[4 * r + 2], buf[4 * r + 3]
        t2 = buf[4 * (r + 1)]
        if t0 == 0 or t1 == 0:
            continue
        ent, edg = pk >> ebits, pk & ((1 << ebits) - 1)
        b_us, x_us = (t1 - t0) / 1e3, (t2 - t1) / 1e3 if t2 else 0.0
        tb += b_us
        tx += x_us
        print(f"{r:>3} {ent:>9} {edg:>11} {le:>12} {le / max(edg, 1):>5.1f} {b_us:>7.1f} {x_us:>8.1f} "
              f"{edg / max(x_us, 1e-9) / 1e3:>8.1f}")
    print(f"sum B {tb:.1f} us, sum X {tx:.1f} us")


if __name__ == "__main__":
    main()
