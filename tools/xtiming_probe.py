"""Per-warp X-phase checkpoints of the sparse (enqueue) path — debug variant
only (build with tools/build_variant.sh xt -DDAWN_XTIMING, run with
DAWN_LIB=.../libdawn_xt.so).

    python tools/xtiming_probe.py [--scale 14 --ef 8 --weights int] [--rounds 1,6,7]
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=14)
    ap.add_argument("--ef", type=int, default=8)
    ap.add_argument("--weights", default="int")
    ap.add_argument("--rounds", default="1,2,6,7,8")
    ap.add_argument("--schedule", default="jacobi")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200.devgen import rmat_device_graph

    dg, _, _ = rmat_device_graph(a.scale, a.ef, weights=a.weights, precision="fp32" if a.weights == "f32" else "auto")
    L = N.lib()
    s = dg.solver(N.F_PROFILE)
    stream = torch.cuda.current_stream().cuda_stream
    fl = N.F_ASYNC if a.schedule == "async" else 0
    for _ in range(3):
        N.check(L.dawn_sssp_begin(s, 0, N.GOVM, fl, stream))
        N.check(L.dawn_sssp_run(s, 0, stream))
    torch.cuda.synchronize()
    buf = np.zeros(16 * 2368 * 6, dtype=np.uint64)
    g = ctypes.c_int(0)
    N.check(L.dawn_solver_cta_profile(s, buf.ctypes.data, 64, ctypes.byref(g), stream))
    buf = buf.reshape(16, 2368, 6).astype(np.int64)
    names = ["filter", "elect", "rows+scan", "reserve", "writes"]
    for r in [int(x) for x in a.rounds.split(",")]:
        b = buf[r]
        ok = (b[:, 0] > 0) & (b[:, 5] > 0)
        if not ok.any():
            print(f"round {r}: no sparse tiles recorded")
            continue
        b = b[ok]
        t0 = b[:, 0].min()
        tot = (b[:, 5] - b[:, 0]) / 1e3
        print(f"round {r}: {ok.sum()} warps; tile total us: median {np.median(tot):.2f} max {tot.max():.2f}; "
              f"first start +0, last end +{(b[:, 5].max() - t0) / 1e3:.2f} us")
        prev = b[:, 0]
        for k, nm in zip(range(1, 6), names):
            cur = b[:, k]
            m = cur > 0
            d = (cur[m] - prev[m]) / 1e3
            if m.any():
                print(f"   {nm:>10}: median {np.median(d):.2f} max {d.max():.2f} us ({m.sum()} warps)")
            prev = np.where(m, cur, prev)


if __name__ == "__main__":
    main()
