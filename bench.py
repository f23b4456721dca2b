#!/usr/bin/env python
"""Benchmark: weighted DAWN (GOVM) SSSP on BASELINE config 2.

Workload (BASELINE.json configs[1]): RMAT scale-22, edge factor 16
(4,194,304 nodes, 67,108,864 edges), float32 weights in [0,1), SSSP from
source 0, one B200.  A "step" is one complete solve (init + all rounds,
device-resident loop).  Under torchrun each rank runs its own replica of the
solve (a single-source SSSP does not shard): value =
sum over ranks of traversed edges / max-over-ranks time  ("scaling": "weak").

Metric: GTEPS = m_reach / t  (Graph500-style: out-edges of every reached
vertex, implementation independent); the relaxed-edge rate R_J / t and the
HBM roofline fraction of the persistent kernel are reported beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

SCALE, EF, SOURCE = 22, 16, 0
PEAKS_FILE = REPO / "MEASURED_PEAKS.json"
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=SCALE)
    ap.add_argument("--ef", type=int, default=EF)
    ap.add_argument("--source", type=int, default=SOURCE)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=120.0, help="seconds for the reference arm's timed steps")
    ap.add_argument("--no-apsp", action="store_true", help="skip the config-3 multi-source leg")
    ap.add_argument("--schedule", choices=["async", "jacobi"], default="async",
                    help="round schedule of the headline solve (the other one is timed beside it)")
    ap.add_argument("--apsp-sources", type=int, default=8192)
    ap.add_argument("--apsp-scale", type=int, default=20)
    ap.add_argument("--dist-backend", default="nccl", help="process-group backend (gloo only for the 1-GPU "
                    "rehearsal of the multi-rank path)")
    ap.add_argument("--device-map", default=None, help="testing: comma list rank->device (e.g. '0' = all on cuda:0)")
    return ap.parse_args()


def hbm_peak():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(args, extra=None):
    cfg = {
        "workload": f"C2: SSSP from source {args.source} on RMAT scale-{args.scale} ef{args.ef} "
                    f"({1 << args.scale} nodes, {args.ef << args.scale} edges), float32 weights U[0,1)",
        "graph": {"kind": "rmat", "scale": args.scale, "edge_factor": args.ef, "abc": [0.57, 0.19, 0.19],
                  "seed": 1, "weights": "float32 U[0,1)", "wseed": 2},
        "algorithm": "govm",
        "source": args.source,
        "parallelism": "replicas (one independent solve per rank)",
    }
    if extra:
        cfg.update(extra)
    return cfg


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", self.gpu_id], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            for name, val in zip(names, r[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference, all host threads)
# ---------------------------------------------------------------------------
def cpu_sources(rp, k: int, source: int):
    import numpy as np

    deg = np.diff(rp)
    cand = np.flatnonzero(deg > 0)
    rng = np.random.default_rng(5)
    extra = rng.choice(cand, size=min(k - 1, cand.size), replace=False) if k > 1 else []
    return [source] + [int(x) for x in extra]


def run_cpu_baseline(host_graph, source: int, threads: int | None = None):
    """k = threads independent reference-order GOVM solves (the reference's own
    parallelism: mssp workers over sources), wall-timed."""
    from oracle import oracle as O

    threads = threads or min(os.cpu_count() or 1, 64)
    srcs = cpu_sources(host_graph.row_ptr, threads, source)
    t0 = time.perf_counter()
    relax, mreach, _ = O.gs_multi(host_graph, srcs, threads=threads)
    dt = time.perf_counter() - t0
    return {
        "value": mreach / dt / 1e9,
        "unit": "GTEPS",
        "cores": threads,
        "kind": "port",
        "sample": f"{len(srcs)} reference-order GOVM solves (source {source} + {len(srcs) - 1} seeded sources with "
                  f"out-degree>=1) on {threads} threads, wall {dt:.2f} s; C restatement of solver.py:212-399 "
                  f"(oracle/dawn_oracle.c), the reference itself is Python and not buildable",
        "relax_gps": relax / dt / 1e9,
        "seconds": dt,
    }


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as O
    from paper_2306_07872_b200.graph import CsrGraph

    threads = min(os.cpu_count() or 1, 64)
    n, m, rp, col, val = O.rmat_csr(args.scale, args.ef, weights="f32", seed=1, wseed=2, threads=threads)
    g = CsrGraph(n=n, m=m, row_ptr=rp, col=col, val=val)
    srcs = cpu_sources(rp, threads, args.source)
    per_step = []
    steps_done = 0
    for _ in range(min(args.warmup, 1)):
        O.gs_multi(g, srcs[:threads], threads=threads)
    budget_end = time.perf_counter() + args.cpu_budget
    mreach_tot = 0
    relax_tot = 0
    while steps_done < args.steps and (steps_done == 0 or time.perf_counter() < budget_end):
        t0 = time.perf_counter()
        r, mr, _ = O.gs_multi(g, srcs, threads=threads)
        per_step.append(time.perf_counter() - t0)
        mreach_tot += mr
        relax_tot += r
        steps_done += 1
    t = sum(per_step)
    value = mreach_tot / t / 1e9
    line = {
        "impl": "reference",
        "metric": "GTEPS (weighted SSSP, Graph500-style m_reach/t)",
        "value": value,
        "unit": "GTEPS",
        "n_gpus": world,
        "steps": steps_done,
        "steps_requested": args.steps,
        "warmup": min(args.warmup, 1),
        "ms_per_step": 1e3 * t / max(steps_done, 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (counter-hash RMAT, generated on the host)",
        "config": workload_config(args, {"parallelism": f"{threads} host threads, one solve per thread"}),
        "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": threads, "kind": "port",
                         "sample": f"each step: {len(srcs)} reference-order GOVM solves (source {args.source} + "
                                   f"seeded sources) on {threads} threads; time budget {args.cpu_budget:.0f} s "
                                   f"caps the step count"},
        "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "relax_gps": relax_tot / t / 1e9,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# config 3: multi-source APSP, sources sharded over the ranks
# ---------------------------------------------------------------------------
def run_apsp(args, rank, world, local):
    """8192 sources on RMAT-20 ef16 (float32 weights), drawn as SURVEY §8(d)
    says (default_rng(5) over vertices with out-degree >= 1, ascending).  The
    timed window runs from the first launch to every float32 result row being
    resident in rank 0's [k][n] tile (max over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2306_07872_b200 import multisource as MS
    from paper_2306_07872_b200.devgen import rmat_device_graph

    dev = torch.device("cuda", local)
    dg, _, deg = rmat_device_graph(args.apsp_scale, 16, weights="f32", precision="fp32", device=local)
    degh = deg.cpu().numpy()
    rng = np.random.default_rng(5)
    cand = np.flatnonzero(degh > 0)
    k = min(args.apsp_sources, cand.size)
    src = sorted(int(x) for x in rng.choice(cand, size=k, replace=False))
    tile = torch.empty((k, dg.n), dtype=torch.float32, device=dev) if rank == 0 else None
    if world == 1:
        MS.mssp_tile(dg, src[:64], out=tile[:64], schedule=args.schedule)  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, stats = MS.mssp_tile(dg, src, out=tile, stats=True, schedule=args.schedule)
        e1.record()
        torch.cuda.synchronize()
        ms, transport = e0.elapsed_time(e1), "local"
    else:
        MS.apsp_sharded(dg, src[: 64 * world], "govm", tile=tile[: 64 * world] if tile is not None else None,
                        schedule=args.schedule)  # warm
        res = MS.apsp_sharded(dg, src, "govm", tile=tile, schedule=args.schedule)
        ms, stats, transport = res.ms_max, res.stats, res.transport
    if rank != 0:
        return None
    R = sum(s.relaxations for s in stats)
    W = sum(s.writes for s in stats)
    b_alg = 12 * R + 16 * (W + k) + 12 * W
    peak, peak_src = hbm_peak()
    t = ms / 1e3
    # spot check: a few rows against single-source solves
    import ctypes
    from paper_2306_07872_b200 import _native as N

    L = N.lib()
    s = dg.solver(0)
    d = torch.empty(dg.n, dtype=torch.float64, device=dev)
    st = N.Stats()
    for i in (0, k // 2, k - 1):
        N.check(L.dawn_sssp(s, src[i], N.GOVM, 0, d.data_ptr(), None, ctypes.byref(st), torch.cuda.current_stream(
            dev).cuda_stream))
        # rows equal the Jacobi single-source solve under either schedule; counters only under Jacobi
        if not torch.equal(d, tile[i].double()) or (args.schedule == "jacobi" and st.relaxations != stats[i].relaxations):
            raise AssertionError(f"APSP row {i} disagrees with the single-source solve")
    return {
        "workload": f"C3: {k} sources on RMAT scale-{args.apsp_scale} ef16 float32 U[0,1) "
                    f"({dg.n} nodes, {dg.m} edges)",
        "metric": "APSP sources/s", "value": k / t, "unit": "sources/s", "n_gpus": world, "ms": ms,
        "sources": k, "batch": MS.BATCH, "transport": transport, "schedule": args.schedule,
        "window": "first launch -> all float32 rows resident in rank 0's [k][n] tile (max over ranks)",
        "relax_gps": R / t / 1e9, "relaxations": R,
        "sssp_equiv_roofline": {"achieved": b_alg / t / 1e9, "peak": peak * world, "unit": "GB/s",
                                "frac": b_alg / t / 1e9 / (peak * world), "peak_source": peak_src,
                                "note": "sum over sources of the single-source algorithmic bytes (12R+16S+12W) with "
                                        "this schedule's own per-source counts; batching 32 sources amortises "
                                        "col/w reads, so this can exceed 1"},
        "rows_checked": 3,
    }


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if args.device_map:
        dm = [int(x) for x in args.device_map.split(",")]
        local = dm[local % len(dm)]
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    red_dev = torch.device("cuda", local) if args.dist_backend == "nccl" else torch.device("cpu")

    from paper_2306_07872_b200 import build as B

    B.build()
    import paper_2306_07872_b200 as P
    from paper_2306_07872_b200 import _native as N
    from paper_2306_07872_b200.devgen import rmat_device_graph

    L = N.lib()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev).cuda_stream

    dg, host, deg = rmat_device_graph(args.scale, args.ef, weights="f32", precision="fp32", device=local,
                                      keep_host=True)
    n = dg.n
    s = dg.solver(0)
    src = args.source
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    K, W = args.steps, args.warmup
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]

    sflag = N.F_ASYNC if args.schedule == "async" else 0

    def step(e=None, flags=None):
        flush.zero_()  # evict L2 outside the timed events
        if e is not None:
            e[0].record()
        N.check(L.dawn_sssp_begin(s, src, N.GOVM, sflag if flags is None else flags, stream))
        if e is not None:
            e[1].record()
        N.check(L.dawn_sssp_run(s, 0, stream))
        if e is not None:
            e[2].record()

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    gpu_id = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    sampler = ClockSampler(gpu_id)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(K):
        step(ev[i])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # keep the GPU busy a little longer so the clock sampler sees the load
    t_end = time.perf_counter() + 0.5
    while time.perf_counter() < t_end:
        step()
        torch.cuda.synchronize()
    clocks = sampler.stop()

    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    kern_ms = [b.elapsed_time(c) for a, b, c in ev]
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())

    # results of the last solve: counters + reached edges
    st = N.Stats()
    dist_dev = torch.empty(n, dtype=torch.float64, device=dev)
    N.check(L.dawn_solver_result(s, dist_dev.data_ptr(), None, ctypes_byref(st), stream))
    fin = torch.isfinite(dist_dev)
    m_reach = int(deg[fin].sum().item())
    R, Wr, steps_run = int(st.relaxations), int(st.writes), int(st.outer_steps)
    import ctypes

    wl = (ctypes.c_uint64 * 6)()
    N.check(L.dawn_solver_worklist_stats(s, wl, stream))
    worklist = ({"from_round": int(wl[0]), "items": int(wl[1]), "warp_batches": int(wl[2]),
                 "span_us": wl[5] / 1e3} if wl[1] else None)
    t_step = tot_ms / K / 1e3
    value = world * m_reach / t_step / 1e9

    # the other schedule, timed the same way (Jacobi: deterministic counters = the oracle's;
    # its R_J, W_J define the algorithmic bytes of the workload)
    oflag = 0 if sflag else N.F_ASYNC
    for _ in range(2):
        step(flags=oflag)
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(max(3, min(K, 20)))]
    for e in ev2:
        step(e, flags=oflag)
    torch.cuda.synchronize()
    o_kern = statistics.mean(b.elapsed_time(c) for a, b, c in ev2) / 1e3
    o_step = statistics.mean(a.elapsed_time(c) for a, b, c in ev2) / 1e3
    st2 = N.Stats()
    N.check(L.dawn_solver_result(s, None, None, ctypes_byref(st2), stream))
    if sflag:
        RJ, WJ = int(st2.relaxations), int(st2.writes)
    else:
        RJ, WJ = R, Wr
    other = {"schedule": "jacobi" if sflag else "async", "ms_per_step": 1e3 * o_step, "kernel_ms": 1e3 * o_kern,
             "value": world * m_reach / o_step / 1e9, "unit": "GTEPS", "relaxations": int(st2.relaxations),
             "writes": int(st2.writes), "rounds": int(st2.outer_steps)}

    # roofline of the persistent kernel (algorithmic bytes):
    # B_alg = 12 R_J + 16 (W_J + 1) + 12 W_J from the snapshot-Jacobi counts
    b_alg = 12 * RJ + 16 * (WJ + 1) + 12 * WJ
    b_act = 12 * R + 16 * (Wr + 1) + 12 * Wr  # the bytes this schedule's own work implies
    t_kern = statistics.mean(kern_ms) / 1e3
    peak, peak_src = hbm_peak()
    achieved = b_alg / t_kern / 1e9
    traffic = None
    prof = REPO / "profiles" / "r01_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end to end through the C ABI with HOST buffers (the reference-facing call) ----
    # every step: the CsrGraph arrays in the reference's layout (int64 row_ptr,
    # int64 col, float64 val; pinned host memory) go to the device
    # (dawn_graph_create converts them in place over PCIe), the solve runs, the
    # float64 distances come back to pinned host memory, and the graph is freed.
    e2e = None
    e2e_resident = None
    if host is not None:
        import ctypes as C

        rp_h = torch.from_numpy(np.array(host.row_ptr)).pin_memory()
        col_h = torch.from_numpy(np.array(host.col)).pin_memory()
        val_h = torch.from_numpy(np.array(host.val)).pin_memory()
        out_h = torch.empty(n, dtype=torch.float64).pin_memory()
        m_edges = int(host.m)
        st_e = N.Stats()

        def e2e_step():
            h = C.c_void_p()
            N.check(L.dawn_graph_create(local, n, m_edges, rp_h.data_ptr(), col_h.data_ptr(), val_h.data_ptr(),
                                        N.F32, 0, C.byref(h)))
            sv = C.c_void_p()
            N.check(L.dawn_solver_create(h, 0, C.byref(sv)))
            N.check(L.dawn_sssp(sv, src, N.GOVM, sflag, out_h.data_ptr(), None, C.byref(st_e), stream))
            N.check(L.dawn_solver_destroy(sv))
            N.check(L.dawn_graph_destroy(h))

        e2e_step()  # warm (context, module load)
        torch.cuda.synchronize()
        KE = max(3, min(K, 5))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(KE):
            e2e_step()
        torch.cuda.synchronize()
        t_e2e = (time.perf_counter() - t0) / KE
        if world > 1:
            tt = torch.tensor([t_e2e], device=red_dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        h2d = 8 * (n + 1) + 16 * m_edges
        e2e = {"value": world * m_reach / t_e2e / 1e9, "unit": "GTEPS", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8 * n + 48, "ms_per_step": 1e3 * t_e2e, "steps": KE,
               "note": "C ABI with host buffers per step: dawn_graph_create from pinned int64/int64/float64 CSR "
                       "(reference CsrGraph layout, read in place over PCIe) + dawn_solver_create + dawn_sssp with "
                       "float64 distances into pinned host memory + destroy; wall clock, max over ranks"}
        if not np.array_equal(np.isfinite(out_h.numpy()), fin.cpu().numpy()):
            raise AssertionError("C-ABI result disagrees with the timed device result")
        # resident graph through the Python API (upload cached, as the reference holds its CsrGraph)
        for _ in range(3):  # warm, in the timed loop's pattern (the result pool reaches its steady state)
            dv, _, _st = P.govm_sssp(host, src, precision="fp32", schedule=args.schedule)
        torch.cuda.synchronize()
        KR = max(3, min(K, 20))
        t0 = time.perf_counter()
        for _ in range(KR):
            dv, _, _st = P.govm_sssp(host, src, precision="fp32", schedule=args.schedule)
        t_res = (time.perf_counter() - t0) / KR
        e2e_resident = {"value": world * m_reach / t_res / 1e9, "unit": "GTEPS", "ms_per_step": 1e3 * t_res,
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8 * n + 48,
                        "note": f"P.govm_sssp(CsrGraph, 0, precision='fp32', schedule='{args.schedule}'), graph "
                                "upload cached by identity"}
        if not np.array_equal(np.isfinite(dv.dist), fin.cpu().numpy()):
            raise AssertionError("public-API result disagrees with the timed device result")

    apsp = None
    if not args.no_apsp:
        apsp = run_apsp(args, rank, world, local)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and host is not None:
        cpu = run_cpu_baseline(host, src)

    line = {
        "metric": "GTEPS (weighted SSSP, Graph500-style m_reach/t)",
        "value": value,
        "unit": "GTEPS",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": tot_ms / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (counter-hash RMAT generated on the device; no dataset)",
        "config": workload_config(args, {"l2": "flushed between steps (256 MiB write outside the timed events)",
                                         "precision": "fp32 (opt-in, <=1e-6 relative vs the fp64 reference)"}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": "dawn_persistent<float,uint32,wide>" + (" + dawn_worklist tail" if sflag else ""),
                     "bytes_alg": b_alg, "kernel_ms": 1e3 * t_kern,
                     "bytes_formula": "12*R_J + 16*(W_J+1) + 12*W_J with the snapshot-Jacobi counts R_J, W_J "
                                      "(BASELINE.md §2; col+w+dist per relax, row_ptr+frontier per scan, "
                                      "dist+frontier per write)",
                     "achieved_own_work": b_act / t_kern / 1e9, "frac_own_work": b_act / t_kern / 1e9 / peak,
                     "own_work_note": "the same formula with this schedule's own R, W"},
        "schedule": {"headline": args.schedule,
                     "note": "async: frontier rows relaxed with their live distance (as the reference's in-place "
                             "order); identical distances, fewer relaxations, counters timing-dependent. jacobi: "
                             "round-start snapshots, counters deterministic and equal to the oracle",
                     "other": other},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_resident": e2e_resident,
        "apsp": apsp,
        # per step: dawn_begin_solve + dawn_persistent (+ dawn_worklist under the async schedule)
        "gpu_launches": (3 if sflag else 2) * K,
        "clocks": clocks,
        "relax_gps": world * R / t_step / 1e9,
        "worklist": worklist,
        "solve": {"rounds": steps_run, "relaxations": R, "writes": Wr, "first_discoveries": int(st.first_discoveries),
                  "m_reach": m_reach, "n": n, "m": dg.m},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ctypes_byref(x):
    import ctypes

    return ctypes.byref(x)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
