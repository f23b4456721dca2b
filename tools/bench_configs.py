"""Measure and parity-check every BASELINE configuration on one GPU.

    python tools/bench_configs.py [--only c1,c2,c4,c5a,c5b] [--out profiles/r01_configs.json]

For each config: the device solve through the C ABI (CUDA events, median of
--solves runs, graph resident), the reference-order CPU port timed on the
same graph (bounded; the grid twin where the full size is infeasible), and
parity: bit-exact distances and exact counters against the snapshot-Jacobi
oracle at FULL size (and the reference-order port where it finishes), plus
the negative-cycle verdict.  Configs:

  c1  RMAT-14 ef8, int 1..100, source 0
  c2  RMAT-22 ef16, float32 U[0,1), source 0 (fp32 path; bench.py's headline)
  c4  4096x4096 4-neighbour grid, int 1..100, source 0 (corner)
  c5a RMAT-18 ef16 + Johnson potentials (negative int weights, no cycle)
  c5b c5a + 1 and 4 injected reachable negative cycles, and 1 unreachable
"""
from __future__ import annotations

import argparse
import ctypes
import json
import statistics
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,c4,c5a,c5b")
    ap.add_argument("--solves", type=int, default=5)
    ap.add_argument("--grid", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200 import generators as G
    from paper_2306_07872_b200.device import DeviceGraph
    from paper_2306_07872_b200.devgen import rmat_csr_device
    from paper_2306_07872_b200.graph import CsrGraph

    L = N.lib()
    stream = torch.cuda.current_stream().cuda_stream
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    results = []

    def device_solve(g: CsrGraph, src: int, precision: str, negcheck: bool):
        dg = DeviceGraph.from_csr(g, precision=precision)
        flags = N.F_NEGCHECK if negcheck else 0
        s = dg.solver(flags)
        ts = []
        for _ in range(a.solves):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(L.dawn_sssp_begin(s, src, N.GOVM, flags, stream))
            N.check(L.dawn_sssp_run(s, 0, stream))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        dist = np.empty(g.n, np.float64)
        st = N.Stats()
        N.check(L.dawn_solver_result(s, dist.ctypes.data, None, ctypes.byref(st), stream))
        vt = N.VTYPE_NAMES[dg.vtype]
        # the async schedule on the same graph: time it and check its distances / flag
        ta = []
        for _ in range(a.solves):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(L.dawn_sssp_begin(s, src, N.GOVM, flags | N.F_ASYNC, stream))
            N.check(L.dawn_sssp_run(s, 0, stream))
            e1.record()
            torch.cuda.synchronize()
            ta.append(e0.elapsed_time(e1))
        da = np.empty(g.n, np.float64)
        sa = N.Stats()
        N.check(L.dawn_solver_result(s, da.ctypes.data, None, ctypes.byref(sa), stream))
        same = bool(np.array_equal(da, dist)) and bool(sa.negative_cycle) == bool(st.negative_cycle) and \
            int(sa.first_discoveries) == int(st.first_discoveries)
        if not bool(st.negative_cycle) and not same:
            raise AssertionError("async schedule disagrees with the Jacobi solve")
        async_rec = {"async_ms_median": statistics.median(ta), "async_relaxations": int(sa.relaxations),
                     "async_equal_to_jacobi": same}
        dg.close()
        return statistics.median(ts), ts, dist, st, vt, async_rec

    def record(name, g, src, ms, ts, dist, st, vt, async_rec, parity, cpu=None, extra=None):
        deg = np.diff(g.row_ptr)
        m_reach = int(deg[np.isfinite(dist)].sum())
        R, W = int(st.relaxations), int(st.writes)
        vb = 4 if vt in ("int32", "float32") else 8
        per = 12 if vb == 4 else 20
        b_alg = per * R + (16 if vb == 4 else 20) * (W + 1) + per * W
        rec = {"config": name, "n": g.n, "m": g.m, "source": src, "vtype": vt, "ms_median": ms,
               "ms_all": [round(x, 4) for x in ts], "rounds": int(st.outer_steps), "relaxations": R, "writes": W,
               "first_discoveries": int(st.first_discoveries), "negative_cycle": bool(st.negative_cycle),
               "early_exit": bool(st.early_exit), "gteps_mreach": m_reach / ms / 1e6,
               "relax_gps": R / ms / 1e6, "roofline_frac": b_alg / (ms / 1e3) / 1e9 / hbm,
               "us_per_round": 1e3 * ms / max(int(st.outer_steps), 1), "parity": parity, "cpu_baseline": cpu}
        rec.update(async_rec)
        rec["async_gteps_mreach"] = m_reach / async_rec["async_ms_median"] / 1e6
        if extra:
            rec.update(extra)
        results.append(rec)
        print(json.dumps(rec), flush=True)

    def rmat_host(scale, ef, weights):
        n, m, rp, col, val = rmat_csr_device(scale, ef, weights=weights)
        g = CsrGraph(n=n, m=m, row_ptr=rp.cpu().numpy(), col=col.cpu().numpy(), val=val.cpu().numpy())
        del rp, col, val
        torch.cuda.empty_cache()
        return g

    def cpu_time(g, src, budget_s=60.0):
        t0 = time.perf_counter()
        d, _, o = O.gs_sssp(g, src, "govm")
        dt = time.perf_counter() - t0
        return d, o, {"seconds": dt, "cores": 1, "kind": "port",
                      "sample": "one reference-order govm solve (C restatement of solver.py:324-399)",
                      "relax_per_s": o["relaxations"] / dt}

    only = set(a.only.split(","))
    if "c1" in only:
        g = rmat_host(14, 8, "int")
        ms, ts, dist, st, vt, ar = device_solve(g, 0, "auto", False)
        od, _, o = O.jacobi_sssp(g, 0, "govm", vtype=vt)
        gd, go, cpu = cpu_time(g, 0)
        parity = {"dist_vs_jacobi_oracle": bool(np.array_equal(dist, od)),
                  "counters_vs_jacobi_oracle": (st.relaxations, st.writes, st.outer_steps) ==
                  (o["relaxations"], o["writes"], o["outer_steps"]),
                  "dist_vs_reference_order_port": bool(np.array_equal(dist, gd))}
        record("c1: RMAT-14 ef8 int 1..100", g, 0, ms, ts, dist, st, vt, ar, parity, cpu)
    if "c2" in only:
        g = rmat_host(22, 16, "f32")
        ms, ts, dist, st, vt, ar = device_solve(g, 0, "fp32", False)
        od, _, o = O.jacobi_sssp(g, 0, "govm", vtype="float32")
        gd, go, cpu = cpu_time(g, 0)
        fin = np.isfinite(gd)
        rel = float(np.max(np.abs(dist[fin] - gd[fin]) / np.maximum(np.abs(gd[fin]), 1e-30))) if fin.any() else 0.0
        parity = {"dist_vs_jacobi_oracle_fp32": bool(np.array_equal(dist, od)),
                  "counters_vs_jacobi_oracle": (st.relaxations, st.writes, st.outer_steps) ==
                  (o["relaxations"], o["writes"], o["outer_steps"]),
                  "reached_set_vs_reference_order_port": bool(np.array_equal(np.isfinite(dist), fin)),
                  "max_rel_err_vs_fp64_reference_order": rel, "tolerance": 1e-6}
        record("c2: RMAT-22 ef16 fp32 U[0,1)", g, 0, ms, ts, dist, st, vt, ar, parity, cpu)
        del g
    if "c4" in only:
        k = a.grid
        g = G.grid_graph(k, k)
        ms, ts, dist, st, vt, ar = device_solve(g, 0, "auto", False)
        t0 = time.perf_counter()
        od, _, o = O.jacobi_sssp(g, 0, "govm", vtype=vt)
        t_or = time.perf_counter() - t0
        parity = {"dist_vs_jacobi_oracle": bool(np.array_equal(dist, od)),
                  "counters_vs_jacobi_oracle": (st.relaxations, st.writes, st.outer_steps) ==
                  (o["relaxations"], o["writes"], o["outer_steps"])}
        # reference-order port on the 1024^2 twin (full size is hours of CPU)
        tw = G.grid_graph(1024, 1024)
        _, _, _, stw, _, _ = device_solve(tw, 0, "auto", False)
        gd, go, cpu = cpu_time(tw, 0)
        twd = np.empty(tw.n)
        dgt = DeviceGraph.from_csr(tw)
        st2 = N.Stats()
        N.check(L.dawn_sssp(dgt.solver(0), 0, N.GOVM, 0, twd.ctypes.data, None, ctypes.byref(st2), stream))
        dgt.close()
        parity["twin_1024_dist_vs_reference_order_port"] = bool(np.array_equal(twd, gd))
        cpu["sample"] = "reference-order govm on the 1024x1024 twin (full 4096^2 is hours on one core)"
        record(f"c4: {k}x{k} grid int 1..100", g, 0, ms, ts, dist, st, vt, ar, parity, cpu,
               {"jacobi_oracle_seconds": t_or})
        del g
    if "c5a" in only or "c5b" in only:
        base, pot = G.johnson_reweight(rmat_host(18, 16, "int"), pseed=3)
        if "c5a" in only:
            ms, ts, dist, st, vt, ar = device_solve(base, 0, "auto", True)
            od, _, o = O.jacobi_sssp(base, 0, "govm", vtype=vt, negcheck=True)
            gd, go, cpu = cpu_time(base, 0)
            parity = {"dist_vs_jacobi_oracle": bool(np.array_equal(dist, od)),
                      "counters_vs_jacobi_oracle": (st.relaxations, st.writes, st.outer_steps) ==
                      (o["relaxations"], o["writes"], o["outer_steps"]),
                      "dist_vs_reference_order_port": bool(np.array_equal(dist, gd)),
                      "negative_edges": int((base.val < 0).sum())}
            record("c5a: RMAT-18 ef16 Johnson-negative int, no cycle", base, 0, ms, ts, dist, st, vt, ar, parity, cpu)
        if "c5b" in only:
            for kc, reach in ((1, True), (4, True), (1, False)):
                cg = G.inject_cycles(base, kc, source=0, seed=7, reachable=reach)
                ms, ts, dist, st, vt, ar = device_solve(cg, 0, "auto", True)
                od, _, o = O.jacobi_sssp(cg, 0, "govm", vtype=vt, negcheck=True)
                parity = {"flag_expected": reach, "flag_vs_jacobi_oracle": bool(st.negative_cycle) ==
                          bool(o["negative_cycle"]) == reach,
                          "counters_vs_jacobi_oracle": (st.relaxations, st.writes, st.outer_steps) ==
                          (o["relaxations"], o["writes"], o["outer_steps"])}
                record(f"c5b: c5a + {kc} {'reachable' if reach else 'unreachable'} negative cycle(s)", cg, 0, ms, ts,
                       dist, st, vt, ar, parity, None,
                       {"note": "early exit by the predecessor-graph cycle check; the reference runs its n-round "
                                "cap (n = 262144 rounds)"})
    if a.out:
        Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
