import sys, ctypes, statistics
sys.path.insert(0, '.')
import torch
from paper_2306_07872_b200 import _native as N, generators as G
from paper_2306_07872_b200.device import DeviceGraph
L = N.lib(); stream = torch.cuda.current_stream().cuda_stream
for name, g in [("c1", G.rmat_graph(14, 8, weights="int"))]:
    dg = DeviceGraph.from_csr(g, precision="auto")
    for cl in (0, 16):
        s = dg.solver(0)
        if cl == 0: N.check(L.dawn_solver_tune(s, b"small_graph", 0.0))
        else:
            N.check(L.dawn_solver_tune(s, b"small_graph", 1.0)); N.check(L.dawn_solver_tune(s, b"small_cluster", float(cl)))
        for fl in (0, N.F_ASYNC):
            ts = []
            for i in range(12):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); N.check(L.dawn_sssp_begin(s, 0, N.GOVM, fl, stream)); N.check(L.dawn_sssp_run(s, 0, stream)); e1.record()
                torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            print(name, "cluster" if cl else "persistent", cl, "async" if fl else "jacobi", round(statistics.median(ts[2:]) * 1e3, 1), "us")
    dg.close()
