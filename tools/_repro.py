import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2306_07872_b200 as P
from paper_2306_07872_b200 import multisource as MS
rng = np.random.default_rng(100)
n = int(rng.integers(2, 600)); m = int(rng.integers(0, 8 * n))
u, v = rng.integers(0, n, m), rng.integers(0, n, m)
w = rng.integers(0, 40, m).astype(float)
g = P.csr_from_arrays(n, u, v, w)
src = [int(x) for x in rng.integers(0, n, 1)]
print(n, m, src)
tile, stats = MS.mssp_tile(g, src, "govm")
print("ok", stats[0])
