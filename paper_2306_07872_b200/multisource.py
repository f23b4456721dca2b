"""Device-resident multi-source / APSP driver.

The reference's ``mssp`` / ``apsp`` (solver.py:426-495) run one Python solve
per source on a fork pool and pickle float64 rows back to the parent.  Here:

* :func:`mssp_tile` — one GPU: the batched kernel (``dawn_mssp_batch``,
  32 sources per pass) writes a device-resident ``[k][n]`` tile, row ``i``
  = distances from ``sources[i]`` (float64, or float32 for float32 graphs).
  Graphs the batched kernel does not take (negative weights, predecessors)
  run one persistent solve per source — still on the GPU.
* :func:`apsp_sharded` — one process per GPU (torchrun): the graph is
  replicated in every HBM, source batches are dealt round-robin over ranks
  (batch ``b`` -> rank ``b % world``), and every rank delivers its rows into
  the root rank's tile in source order.  Transport ``"p2p"``: the root's
  tile is mapped into every rank through CUDA IPC and rows travel as
  copy-engine peer copies over NVLink on a side stream, overlapped with the
  next batch's kernel (no SMs taken from the persistent kernel).
  ``"collective"``: ``torch.distributed`` point-to-point (NCCL, or gloo on
  CPU) after the compute.  Stats are gathered as host objects; the
  ``negative_cycle`` flags travel with them.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as N
from .device import DeviceGraph, device_graph

BATCH = 32  # sources per batched pass (warp lanes)

__all__ = ["BATCH", "batch_supported", "mssp_tile", "apsp_sharded", "shard_batches", "ShardedResult"]


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
# sharding over ranks
# ---------------------------------------------------------------------------
def shard_batches(k: int, world: int, batch: int = BATCH) -> list[list[tuple[int, int]]]:
    """Round-robin deal of source batches: rank r gets [(lo, hi), ...] with
    batch b = [b*batch, min(k, (b+1)*batch)) assigned to rank b % world."""
    out: list[list[tuple[int, int]]] = [[] for _ in range(world)]
    for b, lo in enumerate(range(0, k, batch)):
        out[b % world].append((lo, min(k, lo + batch)))
    return out


@dataclass
class ShardedResult:
    tile: object | None          # root: [k][n] tensor, rows in source order; others: None
    stats: list | None           # root: list[SolveStats] in source order
    ms: float                    # this rank's device time (first launch -> rows delivered)
    ms_max: float                # max over ranks
    transport: str
    batches: int                 # batches this rank solved


def _p2p_possible(root_dev: int, my_dev: int) -> bool:
    import torch

    if root_dev == my_dev:
        return True
    try:
        return bool(torch.cuda.can_device_access_peer(my_dev, root_dev))
    except Exception:
        return False


def apsp_sharded(g, sources: Sequence[int], algo: str = "govm", *, precision: str | None = None,
                 group=None, root: int = 0, out_dtype=None, transport: str = "auto",
                 solve_fn: Callable | None = None, tile=None, ring: int = 3,
                 schedule: str | None = None) -> ShardedResult:
    """Multi-source solve sharded over the ranks of ``group`` (one process per GPU).

    Every rank must call it with the same ``g`` (replicated) and ``sources``.
    ``solve_fn(lo, hi) -> (rows [hi-lo][n] tensor, list[SolveStats])``
    replaces the device solve (tests drive the host logic with it on gloo).
    ``tile``: optional preallocated root tile ``[k][n]`` (reused across calls).
    """
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
    mine = shard_batches(k, world)[rank]

    if transport == "auto":
        transport = "p2p" if on_gpu else "collective"
    if transport == "p2p":
        # every rank must be able to reach the root's HBM; agree on it
        rdev = [dev.index if on_gpu else -1]
        dist.broadcast_object_list(rdev, src=root, group=group)
        ok = torch.tensor([1 if on_gpu and rdev[0] >= 0 and _p2p_possible(rdev[0], dev.index) else 0],
                          device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            transport = "collective"

    if rank == root and tile is None:
        tile = torch.empty((k, n), dtype=out_dtype, device=dev)

    def solve(lo, hi, out_rows):
        if solve_fn is not None:
            rows, st = solve_fn(lo, hi)
            out_rows.copy_(rows)
            return st
        _, st = mssp_tile(dg, src[lo:hi], algo, out=out_rows, out_dtype=out_dtype, stats=True, schedule=schedule)
        return st

    stats_local: list[tuple[int, list]] = []
    t0 = t1 = None
    if on_gpu:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
    dist.barrier(group=group)
    if on_gpu:
        torch.cuda.synchronize(dev)
        t0.record()

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
        for i, (lo, hi) in enumerate(mine):
            if rank == root:
                stats_local.append((lo, solve(lo, hi, tile[lo:hi])))
                continue
            slot = i % ring
            if ring_done[slot] is not None:
                torch.cuda.current_stream(dev).wait_event(ring_done[slot])
            buf = ring_bufs[slot][: hi - lo]
            stats_local.append((lo, solve(lo, hi, buf)))
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
        # compute everything locally, then point-to-point to the root in batch order
        local = {}
        for lo, hi in mine:
            if rank == root:
                rows = tile[lo:hi]
            else:
                rows = torch.empty((hi - lo, n), dtype=out_dtype, device=dev)
            stats_local.append((lo, solve(lo, hi, rows)))
            local[lo] = rows
        plan = shard_batches(k, world)
        # gloo moves host memory only: stage device rows through the host
        staged = on_gpu and backend != "nccl"
        if rank == root:
            reqs = []
            for r in range(world):
                if r == root:
                    continue
                for lo, hi in plan[r]:
                    buf = torch.empty((hi - lo, n), dtype=out_dtype) if staged else tile[lo:hi]
                    reqs.append((dist.irecv(buf, src=r, group=group), lo, hi, buf))
            for q, lo, hi, buf in reqs:
                q.wait()
                if staged:
                    tile[lo:hi].copy_(buf)
        else:
            reqs = [dist.isend(local[lo].cpu() if staged else local[lo], dst=root, group=group) for lo, _ in mine]
            for q in reqs:
                q.wait()
    if on_gpu:
        t1.record()
        torch.cuda.synchronize(dev)
        ms = t0.elapsed_time(t1)
    else:
        ms = 0.0
    dist.barrier(group=group)  # every rank's rows are resident on the root
    tm = torch.tensor([ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(tm, op=dist.ReduceOp.MAX, group=group)
    gathered = [None] * world if rank == root else None
    dist.gather_object(stats_local, gathered, dst=root, group=group)
    stats = None
    if rank == root:
        stats = [None] * k
        for part in gathered:
            for lo, sts in part:
                stats[lo:lo + len(sts)] = sts
    return ShardedResult(tile=tile if rank == root else None, stats=stats, ms=ms, ms_max=float(tm.item()),
                         transport=transport, batches=len(mine))
