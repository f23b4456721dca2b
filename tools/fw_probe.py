"""Timing of the device Floyd–Warshall (F4) against the reference-style NumPy loop.

    python tools/fw_probe.py [--n 2000] [--numpy-steps 20]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[1000, 2000, 4000])
    ap.add_argument("--numpy-steps", type=int, default=20, help="NumPy steps timed (extrapolated to n)")
    a = ap.parse_args()
    import numpy as np

    import paper_2306_07872_b200 as P

    for n in a.n:
        rng = np.random.default_rng(n)
        m = 8 * n
        g = P.csr_from_arrays(n, rng.integers(0, n, m), rng.integers(0, n, m), rng.uniform(0, 1, m))
        P.floyd_warshall_apsp(g, cap=n)  # warm
        t0 = time.perf_counter()
        fw = P.floyd_warshall_apsp(g, cap=n)
        t = time.perf_counter() - t0
        mat = np.array(fw.matrix)
        t1 = time.perf_counter()
        for k in range(a.numpy_steps):
            np.minimum(mat, mat[:, k:k + 1] + mat[k:k + 1, :], out=mat)
        tn = (time.perf_counter() - t1) / a.numpy_steps * n
        print(f"n={n}: device {t * 1e3:.1f} ms (incl. upload + {8 * n * n / 1e6:.0f} MB matrix to pinned host), "
              f"{n ** 3 / t / 1e9:.1f} G min-plus/s; NumPy loop ~{tn:.1f} s (extrapolated from "
              f"{a.numpy_steps} steps)")


if __name__ == "__main__":
    main()
