"""Device-resident multi-source / APSP driver.

The reference's ``mssp`` / ``apsp`` (solver.py:426-495) run one Python solve
per source on a fork pool and pickle float64 rows back to the parent.  Here:

* :func:`mssp_tile` — one GPU: the batched kernel (``dawn_mssp_batch``,
  32 sources per pass) writes a device-resident ``[k][n]`` tile, row ``i``
  = distances from ``sources[i]`` (float64, or float32 for float32 graphs).
  Graphs the batched kernel does not take (negative weights, predecessors)
  run one persistent solve per source — still on the GPU.
* :func:`apsp_sharded` — one process per GPU (torchrun): the graph is
  replicated in every HBM, ranks claim source batches dynamically from a
  group-wide cursor (per-source cost varies by orders of magnitude), and
  every rank delivers its rows into the root rank's tile at the batch's
  offset, so the tile is in source order.  Transport ``"p2p"``: the root's
  tile is mapped into every rank through CUDA IPC and rows travel as
  copy-engine peer copies over NVLink on a side stream, overlapped with the
  next batch's kernel (no SMs taken from the persistent kernel).
  ``"collective"``: ``torch.distributed`` point-to-point (NCCL, or gloo on
  CPU) after the compute.  Per-source counters and the ``negative_cycle``
  flags travel in one ``all_reduce``; per-rank load in one ``all_gather``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as N
from .device import DeviceGraph, device_graph

BATCH = 32  # sources per batched pass (warp lanes)

__all__ = ["BATCH", "batch_supported", "mssp_tile", "apsp_sharded", "batch_bounds", "shard_batches", "BatchCursor",
           "ShardedResult"]


def _algo_id(algo: str) -> int:
    return {"govm": N.GOVM, "gsvm": N.GSVM}[algo.lower()]


def batch_supported(dg: DeviceGraph, algo: str = "govm", flags: int = 0) -> bool:
    """True when ``dawn_mssp_batch`` takes this graph (no negative weight, n >= 2)."""
    out = ctypes.c_int(0)
    with dg.lock:
        N.check(N.lib().dawn_batch_supported(dg.solver(0), _algo_id(algo), flags, ctypes.byref(out)))
    return bool(out.value)


def _stats_list(arr, k):
    from .solver import _stats_from_native

    return [_stats_from_native(arr[i]) for i in range(k)]


def mssp_tile(g, sources: Sequence[int], algo: str = "govm", *, precision: str | None = None,
              out=None, out_dtype=None, stats: bool = True, device: int | None = None,
              schedule: str | None = None):
    """Distances from every source into a device tensor tile ``[k][n]``.

    ``out``: optional preallocated CUDA tensor view ``[k][ld >= n]`` (row
    stride ``ld``) of dtype ``out_dtype``; float64 by default, float32
    allowed for float32 graphs.  Returns ``(tile, stats)`` with ``stats`` a
    list of :class:`SolveStats` (or None when ``stats=False``, in which case
    the call is asynchronous on the current stream).  ``schedule``:
    ``jacobi`` / ``async`` as in :func:`gsvm_sssp`.
    """
    import torch

    from .solver import _schedule_flag

    sflag = _schedule_flag(schedule)

    dg = device_graph(g, device=device, precision=precision)
    src = np.ascontiguousarray([int(s) for s in sources], dtype=np.int64)
    k, n = int(src.size), dg.n
    for s in src.tolist():
        if not 0 <= s < n:
            raise ValueError(f"source {s} out of range for n={n}")
    if out_dtype is None:
        out_dtype = out.dtype if out is not None else torch.float64
    if out_dtype not in (torch.float64, torch.float32):
        raise ValueError("out_dtype must be torch.float64 or torch.float32")
    if out_dtype == torch.float32 and dg.vtype != N.F32:
        raise ValueError("float32 tiles need a float32 graph (precision='fp32')")
    dev = torch.device("cuda", dg.device)
    if out is None:
        out = torch.empty((k, n), dtype=out_dtype, device=dev)
    if out.dim() != 2 or out.shape[0] != k or out.shape[1] < n or out.stride(1) != 1 or out.dtype != out_dtype:
        raise ValueError("out must be a [k][>=n] row-major view of out_dtype")
    ld = out.stride(0) if k > 1 else max(n, out.shape[1])
    vt = N.F64 if out_dtype == torch.float64 else N.F32
    algo_id = _algo_id(algo)
    st_arr = (N.Stats * max(k, 1))() if stats else None
    with dg.lock:
        s = dg.solver(0)
        stream = dg.stream()
        sup = ctypes.c_int(0)
        N.check(N.lib().dawn_batch_supported(s, algo_id, 0, ctypes.byref(sup)))
        if sup.value:
            N.check(N.lib().dawn_mssp_batch(s, src.ctypes.data, k, algo_id, sflag, out.data_ptr(), vt, ld,
                                            ctypes.addressof(st_arr) if stats else None, stream))
        else:
            # negative weights: one persistent solve per source (integer graphs keep the
            # early negative-cycle exit), float64 rows
            flags = (N.F_NEGCHECK if dg.vtype in (N.I32, N.I64) else 0) | sflag
            s2 = dg.solver(flags)
            row = out if vt == N.F64 else torch.empty((k, n), dtype=torch.float64, device=dev)
            for i in range(k):
                N.check(N.lib().dawn_sssp(s2, int(src[i]), algo_id, flags, row[i].data_ptr(), None,
                                          ctypes.byref(st_arr[i]) if stats else None, stream))
            if row is not out:
                out[:, :n].copy_(row)
    return out, (_stats_list(st_arr, k) if stats else None)


# ---------------------------------------------------------------------------
# sharding over ranks: dynamic batch claiming
# ---------------------------------------------------------------------------
def batch_bounds(k: int, batch: int = BATCH) -> list[tuple[int, int]]:
    """Batch b = sources [b*batch, min(k, (b+1)*batch))."""
    return [(lo, min(k, lo + batch)) for lo in range(0, k, batch)]


def shard_batches(k: int, world: int, batch: int = BATCH) -> list[list[tuple[int, int]]]:
    """Static round-robin deal (batch b -> rank b % world); kept as the
    ``claim="static"`` plan and for comparison with the dynamic cursor."""
    out: list[list[tuple[int, int]]] = [[] for _ in range(world)]
    for b, lohi in enumerate(batch_bounds(k, batch)):
        out[b % world].append(lohi)
    return out


class BatchCursor:
    """A group-wide atomic batch counter: ``claim()`` returns the next
    unclaimed batch index (>= the batch count once all are taken).

    The counter lives in the process group's key-value store (rank 0's
    TCPStore), so a claim is one ``add`` round trip (~0.1 ms) against a
    ~8 ms batch solve; ranks that draw cheap sources simply come back sooner.
    This is the reference's chunked pool hand-out (solver.py:453-457,
    :487-494) across processes.  ``static`` deals ``b % world`` instead."""

    _calls = 0

    def __init__(self, nbatches: int, group=None, static: bool = False):
        import torch.distributed as dist

        self.nbatches = nbatches
        self.static = static
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        BatchCursor._calls += 1  # collective call order is the same on every rank
        self.key = f"dawn/apsp/{BatchCursor._calls}"
        self._next_static = self.rank
        self.store = None
        if not static:
            from torch.distributed import distributed_c10d as c10d

            self.store = c10d._get_default_store()

    def claim(self) -> int:
        if self.static:
            b = self._next_static
            self._next_static += self.world
            return b
        return int(self.store.add(self.key, 1)) - 1


# native counters carried per source through the stats all-reduce
_STAT_FIELDS = ("outer_steps", "relaxations", "writes", "first_discoveries", "multi_written", "negative_cycle",
                "early_exit")


def _stats_to_row(st) -> list[int]:
    """A SolveStats (or native Stats) as the int64 row the all-reduce carries."""
    if hasattr(st, "multi_written"):
        return [int(getattr(st, f)) for f in _STAT_FIELDS]
    fd = int(st.first_discoveries)
    multi = int(round(st.updated_ratio * max(fd, 1)))
    return [int(st.outer_steps), int(st.relaxations), int(st.writes), fd, multi, int(bool(st.negative_cycle)), 0]


def _solve_stats_from_row(row) -> "object":
    from .solver import _stats_from_native

    st = N.Stats()
    for f, v in zip(_STAT_FIELDS, row):
        setattr(st, f, int(v))
    return _stats_from_native(st)


def _p2p_possible(root_dev: int, my_dev: int) -> bool:
    import torch

    if root_dev == my_dev:
        return True
    try:
        return bool(torch.cuda.can_device_access_peer(my_dev, root_dev))
    except Exception:
        return False


@dataclass
class ShardedResult:
    tile: object | None          # root: [k][n] tensor, rows in source order; others: None
    stats: list | None           # every rank: list[SolveStats] in source order (all-reduced)
    ms: float                    # this rank's device time (first launch -> rows delivered)
    ms_max: float                # max over ranks
    transport: str
    batches: int                 # batches this rank solved
    claimed: list | None = None  # this rank's batch indices, in claim order
    per_rank: list | None = None  # every rank: [{"rank", "batches", "sources", "busy_ms"}]


def apsp_sharded(g, sources: Sequence[int], algo: str = "govm", *, precision: str | None = None,
                 group=None, root: int = 0, out_dtype=None, transport: str = "auto",
                 solve_fn: Callable | None = None, tile=None, ring: int = 3,
                 schedule: str | None = None, claim: str = "dynamic") -> ShardedResult:
    """Multi-source solve sharded over the ranks of ``group`` (one process per GPU).

    Every rank must call it with the same ``g`` (replicated in every HBM) and
    ``sources``.  Batches of :data:`BATCH` sources are claimed dynamically
    from a group-wide cursor (:class:`BatchCursor`; ``claim="static"`` deals
    them round-robin), each rank solves what it claims and delivers the rows
    into the root's ``[k][n]`` tile at the batch's offset, so the tile is in
    source order whatever rank solved a batch.  Per-source counters travel in
    one ``all_reduce(SUM)`` of a ``[k][7]`` int64 tensor (every rank ends with
    all stats; ``negative_cycle`` included), per-rank load in one
    ``all_gather``.  ``solve_fn(lo, hi) -> (rows [hi-lo][n] tensor,
    list[SolveStats-like])`` replaces the device solve (tests drive the host
    logic with it on gloo); ``tile``: optional preallocated root tile.
    """
    import time

    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    src = [int(s) for s in sources]
    k = len(src)
    backend = dist.get_backend(group)
    on_gpu = solve_fn is None
    if on_gpu:
        dg = device_graph(g, precision=precision)
        n = dg.n
        dev = torch.device("cuda", dg.device)
        if out_dtype is None:
            out_dtype = torch.float32 if dg.vtype == N.F32 else torch.float64
    else:
        n = int(g.n)
        dev = torch.device("cpu")
        if out_dtype is None:
            out_dtype = torch.float64
    for s in src:
        if not 0 <= s < n:
            raise ValueError(f"source {s} out of range for n={n}")
    if claim not in ("dynamic", "static"):
        raise ValueError(f"unknown claim mode {claim!r}")
    cdev = dev if backend == "nccl" else torch.device("cpu")  # collectives' device
    bounds = batch_bounds(k)
    cursor = BatchCursor(len(bounds), group, static=(claim == "static"))

    if transport == "auto":
        transport = "p2p" if on_gpu else "collective"
    if transport == "p2p":
        # every rank must be able to reach the root's HBM; agree on it
        rdev = [dev.index if on_gpu else -1]
        dist.broadcast_object_list(rdev, src=root, group=group)
        ok = torch.tensor([1 if on_gpu and rdev[0] >= 0 and _p2p_possible(rdev[0], dev.index) else 0],
                          device=cdev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            transport = "collective"

    if rank == root and tile is None:
        tile = torch.empty((k, n), dtype=out_dtype, device=dev)

    stat_rows = torch.zeros((max(k, 1), len(_STAT_FIELDS)), dtype=torch.int64)

    def solve(lo, hi, out_rows):
        if solve_fn is not None:
            rows, st = solve_fn(lo, hi)
            out_rows.copy_(rows)
        else:
            _, st = mssp_tile(dg, src[lo:hi], algo, out=out_rows, out_dtype=out_dtype, stats=True,
                              schedule=schedule)
        stat_rows[lo:hi] = torch.tensor([_stats_to_row(x) for x in st], dtype=torch.int64)

    def claims():
        while True:
            b = cursor.claim()
            if b >= len(bounds):
                return
            yield b

    claimed: list[int] = []
    t0 = t1 = None
    if on_gpu:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
    dist.barrier(group=group)
    if on_gpu:
        torch.cuda.synchronize(dev)
        t0.record()
    w0 = time.perf_counter()

    if transport == "p2p":
        # map the root's tile into this process (CUDA IPC) -> copy-engine peer copies
        from torch.multiprocessing.reductions import reduce_tensor

        obj = [reduce_tensor(tile) if rank == root else None]
        dist.broadcast_object_list(obj, src=root, group=group)
        if rank == root:
            remote = tile
        else:
            fn, args = obj[0]
            remote = fn(*args)
        cstream = torch.cuda.Stream(device=dev)
        ring_bufs = [torch.empty((BATCH, n), dtype=out_dtype, device=dev) for _ in range(ring)] if rank != root else []
        ring_done = [None] * len(ring_bufs)
        for i, b in enumerate(claims()):
            lo, hi = bounds[b]
            claimed.append(b)
            if rank == root:
                solve(lo, hi, tile[lo:hi])
                continue
            slot = i % ring
            if ring_done[slot] is not None:
                torch.cuda.current_stream(dev).wait_event(ring_done[slot])
            buf = ring_bufs[slot][: hi - lo]
            solve(lo, hi, buf)
            ready = torch.cuda.Event()
            ready.record()
            with torch.cuda.stream(cstream):
                cstream.wait_event(ready)
                remote[lo:hi].copy_(buf, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cstream)
                ring_done[slot] = ev
        if rank != root:
            cstream.synchronize()
    else:
        # compute what this rank claims, then point-to-point to the root in claim order
        local = {}
        for b in claims():
            lo, hi = bounds[b]
            claimed.append(b)
            rows = tile[lo:hi] if rank == root else torch.empty((hi - lo, n), dtype=out_dtype, device=dev)
            solve(lo, hi, rows)
            local[b] = rows
        plan = [None] * world
        dist.all_gather_object(plan, claimed, group=group)
        # gloo moves host memory only: stage device rows through the host
        staged = on_gpu and backend != "nccl"
        if rank == root:
            reqs = []
            for r in range(world):
                if r == root:
                    continue
                for b in plan[r]:
                    lo, hi = bounds[b]
                    buf = torch.empty((hi - lo, n), dtype=out_dtype) if staged else tile[lo:hi]
                    reqs.append((dist.irecv(buf, src=r, group=group), lo, hi, buf))
            for q, lo, hi, buf in reqs:
                q.wait()
                if staged:
                    tile[lo:hi].copy_(buf)
        else:
            reqs = [dist.isend(local[b].cpu() if staged else local[b], dst=root, group=group) for b in claimed]
            for q in reqs:
                q.wait()
    if on_gpu:
        t1.record()
        torch.cuda.synchronize(dev)
        ms = t0.elapsed_time(t1)
    else:
        ms = 1e3 * (time.perf_counter() - w0)
    dist.barrier(group=group)  # every rank's rows are resident on the root
    tm = torch.tensor([ms], dtype=torch.float64, device=cdev)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX, group=group)
    # per-source counters: each source solved by exactly one rank -> SUM = gather
    st_red = stat_rows.to(cdev)
    dist.all_reduce(st_red, op=dist.ReduceOp.SUM, group=group)
    st_all = st_red.cpu().numpy()
    stats = [_solve_stats_from_row(st_all[i]) for i in range(k)]
    nsrc = sum(bounds[b][1] - bounds[b][0] for b in claimed)
    load = torch.tensor([[rank, len(claimed), nsrc, ms]], dtype=torch.float64, device=cdev)
    loads = [torch.empty_like(load) for _ in range(world)]
    dist.all_gather(loads, load, group=group)
    per_rank = [{"rank": int(x[0, 0]), "batches": int(x[0, 1]), "sources": int(x[0, 2]), "busy_ms": float(x[0, 3])}
                for x in (t.cpu() for t in loads)]
    return ShardedResult(tile=tile if rank == root else None, stats=stats, ms=ms, ms_max=float(tm.item()),
                         transport=transport, batches=len(claimed), claimed=claimed, per_rank=per_rank)
