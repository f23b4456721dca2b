"""Drop-in weighted-DAWN solvers on the GPU (mirror of sparsepath/solver.py).

Public names, signatures, return types and error behaviour follow the
reference (``/root/reference/pkg/src/sparsepath/solver.py``):

  ===================  ==========================  ===============================
  this module          reference                   device path
  ===================  ==========================  ===============================
  ``seed_source``      solver.py:212-250           round 1 of the persistent kernel
  ``gsvm_sssp``        solver.py:265-321           dawn_sssp(algo=GSVM)
  ``govm_sssp``        solver.py:324-399           dawn_sssp(algo=GOVM)
  ``SOLVERS``          solver.py:402               same names
  ``mssp``             solver.py:426-457           dawn_mssp, sources over GPUs
  ``apsp``             solver.py:460-495           dawn_mssp in row blocks -> sink
  ===================  ==========================  ===============================

Semantics.  Distances and the ``negative_cycle`` flag equal the reference's:
both the reference's in-place (Gauss-Seidel) relaxation and the device's
frontier-synchronous (snapshot-Jacobi) rounds converge to the same greatest
fixpoint of ``d[v] = min(d[v], fl(d[u] + w))`` with the source pinned, so
integer and float64 results are bit-identical.  Work counters are reported
under snapshot-Jacobi round semantics: deterministic
across runs, ``workers`` and devices, equal to the reference on its
known-answer fixtures, but not equal to its Gauss-Seidel counts on large
graphs.  ``trace`` and ``record_pred`` run a host-synchronised stepping /
predecessor pass on the device.
"""

from __future__ import annotations

import ctypes
import threading
from concurrent.futures import ThreadPoolExecutor
from ctypes import byref, c_int, c_int64
from dataclasses import dataclass
from math import inf
from typing import Callable, Iterable, Sequence

import numpy as np

from . import _native as N
from . import device as _dev
from .device import DeviceGraph, device_graph

__all__ = [
    "DistanceVector",
    "PredecessorVector",
    "FrontierFlags",
    "SolveStats",
    "AggregateStats",
    "seed_source",
    "gsvm_sssp",
    "govm_sssp",
    "mssp",
    "mssp_stats",
    "apsp",
    "aggregate_stats",
    "format_distance_row",
    "SOLVERS",
]


# ---------------------------------------------------------------------------
# result types (reference solver.py:66-209)
# ---------------------------------------------------------------------------
@dataclass(frozen=True, eq=False)
class DistanceVector:
    """Distances from ``source``; ``inf`` = unreachable (solver.py:66-71)."""

    dist: np.ndarray
    source: int


@dataclass
class PredecessorVector:
    """Shortest-path tree witness (solver.py:74-98).

    ``pred[j]`` is a node whose value produced ``dist[j]`` in the round that
    last lowered ``j`` (the smallest such node id — deterministic; the
    reference keeps the last writer in CSR order).  ``pred[source]`` is None.
    """

    pred: list
    source: int

    def path_to(self, j: int) -> list[int] | None:
        if j != self.source and self.pred[j] is None:
            return None
        path = [j]
        seen = {j}
        node = j
        while node != self.source:
            node = self.pred[node]
            if node is None or node in seen:  # broken chain (negative cycle)
                return None
            seen.add(node)
            path.append(node)
        return path[::-1]


@dataclass
class FrontierFlags:
    """Alg. 2's two frontier vectors (solver.py:101-115); host-side only."""

    current: list
    next: list

    @classmethod
    def empty(cls, n: int) -> "FrontierFlags":
        return cls(current=[False] * n, next=[False] * n)


@dataclass
class SolveStats:
    """Per-solve work counters (solver.py:118-149)."""

    outer_steps: int = 0
    relaxations: int = 0
    writes: int = 0
    first_discoveries: int = 0
    re_updates: int = 0
    mu: float = 0.0
    updated_ratio: float = 0.0
    negative_cycle: bool = False

    def as_dict(self) -> dict:
        return {
            "outer_steps": self.outer_steps,
            "relaxations": self.relaxations,
            "writes": self.writes,
            "first_discoveries": self.first_discoveries,
            "re_updates": self.re_updates,
            "mu": self.mu,
            "updated_ratio": self.updated_ratio,
            "negative_cycle": self.negative_cycle,
        }


@dataclass
class AggregateStats:
    """Counters summed over solves; means over sources that reach a node (solver.py:152-202)."""

    sources: int = 0
    reachable_sources: int = 0
    outer_steps: int = 0
    relaxations: int = 0
    writes: int = 0
    first_discoveries: int = 0
    re_updates: int = 0
    mean_mu: float = 0.0
    mean_updated_ratio: float = 0.0
    negative_cycle: bool = False

    def add(self, s: SolveStats) -> None:
        self.sources += 1
        self.outer_steps += s.outer_steps
        self.relaxations += s.relaxations
        self.writes += s.writes
        self.first_discoveries += s.first_discoveries
        self.re_updates += s.re_updates
        self.negative_cycle = self.negative_cycle or bool(s.negative_cycle)
        if s.first_discoveries > 0:
            self.reachable_sources += 1
            self.mean_mu += s.mu  # running sums until finish()
            self.mean_updated_ratio += s.updated_ratio

    def finish(self) -> "AggregateStats":
        if self.reachable_sources:
            self.mean_mu /= self.reachable_sources
            self.mean_updated_ratio /= self.reachable_sources
        return self

    def as_dict(self) -> dict:
        return {
            "sources": self.sources,
            "reachable_sources": self.reachable_sources,
            "outer_steps": self.outer_steps,
            "relaxations": self.relaxations,
            "writes": self.writes,
            "first_discoveries": self.first_discoveries,
            "re_updates": self.re_updates,
            "mean_mu": self.mean_mu,
            "mean_updated_ratio": self.mean_updated_ratio,
            "negative_cycle": self.negative_cycle,
        }


def aggregate_stats(stats: Iterable[SolveStats]) -> AggregateStats:
    agg = AggregateStats()
    for s in stats:
        agg.add(s)
    return agg.finish()


def _stats_from_native(st: N.Stats) -> SolveStats:
    """``_finalize`` (solver.py:258-262) over the device counters."""
    w, fd = int(st.writes), int(st.first_discoveries)
    denom = max(fd, 1)
    return SolveStats(
        outer_steps=int(st.outer_steps),
        relaxations=int(st.relaxations),
        writes=w,
        first_discoveries=fd,
        re_updates=w - fd,
        mu=w / denom,
        updated_ratio=int(st.multi_written) / denom,
        negative_cycle=bool(st.negative_cycle),
    )


# ---------------------------------------------------------------------------
# argument checks (same messages as the reference)
# ---------------------------------------------------------------------------
def _check_source(g, source: int) -> None:
    if not 0 <= source < g.n:
        raise ValueError(f"source {source} out of range for n={g.n}")


def _normalize_algo(algo: str) -> str:
    name = algo.lower()
    if name not in SOLVERS:
        raise ValueError(f"unknown solver {algo!r}; expected one of {sorted(SOLVERS)}")
    return name


_ALGO = {"govm": N.GOVM, "gsvm": N.GSVM}


def _neg_flags(dg: DeviceGraph) -> int:
    # integer graphs with negative edges: predecessor-graph cycle check gives
    # the cap's verdict early (DESIGN.md §Negative cycles)
    return N.F_NEGCHECK if dg.vtype in (N.I32, N.I64) else 0


# ---------------------------------------------------------------------------
# single-source solves
# ---------------------------------------------------------------------------
def _schedule_flag(schedule: str | None) -> int:
    sch = schedule or _dev.get_default_schedule()
    if sch not in _dev.SCHEDULES:
        raise ValueError(f"unknown schedule {sch!r}; expected one of {list(_dev.SCHEDULES)}")
    return N.F_ASYNC if sch == "async" else 0


_PINNED_LOCK = threading.Lock()
_PINNED_LIVE = [0, 0]       # [result arrays in pooled pinned memory still alive, their bytes]
_PINNED_LIMIT = (4, 1 << 30)
_PINNED_FREE: dict[int, list] = {}  # nbytes -> page-locked blocks (torch uint8 tensors) ready for reuse
_PINNED_KEEP = 4                    # free blocks kept per size


def _pinned_released(nbytes: int, block) -> None:
    with _PINNED_LOCK:
        _PINNED_LIVE[0] -= 1
        _PINNED_LIVE[1] -= nbytes
        free = _PINNED_FREE.setdefault(nbytes, [])
        if len(free) < _PINNED_KEEP:
            free.append(block)


def _host_array(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory from a small pool of reused
    blocks: the device writes results into it at full PCIe speed with no page
    faults (a config-2 distance vector: ~0.6 ms instead of ~7 ms into fresh
    pageable memory), and the block goes back to the pool when the array (and
    every view of it) is gone.  A caller that keeps many results alive gets
    pageable arrays beyond 4 live blocks or 1 GB; single results over 1 GB are
    always pageable (page-locking them would cost more than it saves)."""
    import weakref

    count = int(np.prod(shape)) if isinstance(shape, tuple) else int(shape)
    nbytes = count * np.dtype(dtype).itemsize
    with _PINNED_LOCK:
        if nbytes == 0 or nbytes > (1 << 30) or _PINNED_LIVE[0] >= _PINNED_LIMIT[0] or \
                _PINNED_LIVE[1] + nbytes > _PINNED_LIMIT[1]:
            return np.empty(shape, dtype=dtype)
        free = _PINNED_FREE.get(nbytes)
        block = free.pop() if free else None
        _PINNED_LIVE[0] += 1
        _PINNED_LIVE[1] += nbytes
    if block is None:
        block = _new_pinned_block(nbytes)
    # every view of the result (rows[i], dist[a:b], ...) has ``raw`` as its
    # base, so the block goes back to the pool only when the last view dies
    raw = block.numpy()
    weakref.finalize(raw, _pinned_released, nbytes, block)
    return raw.view(dtype).reshape(shape)


def _new_pinned_block(nbytes: int):
    import torch

    return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)


def _solve(g, source: int, algo: int, record_pred: bool, precision: str | None, schedule: str | None = None):
    _check_source(g, int(source))
    dg = device_graph(g, precision=precision)
    flags = (N.F_PRED if record_pred else 0) | _neg_flags(dg) | _schedule_flag(schedule)
    with dg.lock:
        s = dg.solver(flags)
        dist = _host_array(dg.n)
        pred = np.empty(dg.n, dtype=np.int64) if record_pred else None
        st = N.Stats()
        N.check(N.lib().dawn_sssp(s, int(source), algo, flags, dist.ctypes.data,
                                  pred.ctypes.data if pred is not None else None, byref(st), dg.stream()))
    dv = DistanceVector(dist=dist, source=int(source))
    pv = None
    if record_pred:
        pv = PredecessorVector(pred=[None if p < 0 else int(p) for p in pred.tolist()], source=int(source))
    return dv, pv, _stats_from_native(st)


def _solve_traced(g, source: int, algo: int, record_pred: bool, trace, precision: str | None,
                  schedule: str | None = None):
    """Host-synchronised stepping for the ``trace`` hook (solver.py:328-336, :386-387).

    ``scanned`` for round r is the set lowered in round r-1 and ``written`` the
    set lowered in round r, both ascending — the write stamps on the device
    record the last round that lowered each node.
    """
    _check_source(g, int(source))
    dg = device_graph(g, precision=precision)
    flags = (N.F_PRED if record_pred else 0) | _neg_flags(dg) | _schedule_flag(schedule)
    L = N.lib()
    with dg.lock:
        s = dg.solver(flags)
        stream = dg.stream()
        n = dg.n
        dist = np.empty(n, dtype=np.float64)
        stamp = np.empty(n, dtype=np.uint32)
        rnd, done = c_int64(0), c_int(0)
        N.check(L.dawn_sssp_begin(s, int(source), algo, flags, stream))
        N.check(L.dawn_sssp_advance(s, 1, byref(rnd), byref(done), stream))  # seeding round
        N.check(L.dawn_solver_state(s, None, stamp.ctypes.data, stream))
        prev_written = np.flatnonzero(stamp == 1).tolist()
        last = rnd.value
        while True:
            N.check(L.dawn_sssp_advance(s, 1, byref(rnd), byref(done), stream))
            if rnd.value == last:
                break
            last = rnd.value
            N.check(L.dawn_solver_state(s, dist.ctypes.data, stamp.ctypes.data, stream))
            written = np.flatnonzero(stamp == last).tolist()
            trace(int(last), prev_written, written, dist.tolist())
            prev_written = written
        dist_out = np.empty(n, dtype=np.float64)
        pred = np.empty(n, dtype=np.int64) if record_pred else None
        st = N.Stats()
        N.check(L.dawn_solver_result(s, dist_out.ctypes.data, pred.ctypes.data if pred is not None else None,
                                     byref(st), stream))
    dv = DistanceVector(dist=dist_out, source=int(source))
    pv = None
    if record_pred:
        pv = PredecessorVector(pred=[None if p < 0 else int(p) for p in pred.tolist()], source=int(source))
    return dv, pv, _stats_from_native(st)


def gsvm_sssp(g, source: int, record_pred: bool = False, *, precision: str | None = None,
              schedule: str | None = None):
    """Full-rescan SSSP (Alg. 1; reference solver.py:265-321) on the GPU.

    Returns ``(DistanceVector, PredecessorVector | None, SolveStats)``.
    Extensions: ``precision`` — ``auto``/``fp32``/``fp64``, default from
    :func:`set_default_precision`; ``schedule`` — ``jacobi``/``async``,
    default from :func:`set_default_schedule`.
    """
    return _solve(g, source, N.GSVM, record_pred, precision, schedule)


def govm_sssp(g, source: int, record_pred: bool = False, trace: Callable | None = None, *,
              precision: str | None = None, schedule: str | None = None):
    """Frontier SSSP (Alg. 2; reference solver.py:324-399) on the GPU.

    ``trace(step, scanned_nodes, written_nodes, distance_snapshot)`` is called
    after every round from step 2 on, as in the reference.  ``precision`` and
    ``schedule`` as in :func:`gsvm_sssp`.
    """
    if trace is not None:
        return _solve_traced(g, source, N.GOVM, record_pred, trace, precision, schedule)
    return _solve(g, source, N.GOVM, record_pred, precision, schedule)


def seed_source(g, source: int, alpha: list, delta: list, stats: SolveStats | None = None,
                pred: list | None = None, write_counts: list | None = None):
    """Round 1 of a solve (reference solver.py:212-250), executed on the device.

    Expects ``alpha`` all-infinite except ``alpha[source] == 0`` and ``delta``
    all-false; updates them in place and returns ``(alpha, delta)``.
    """
    _check_source(g, int(source))
    dg = device_graph(g)
    L = N.lib()
    n = dg.n
    with dg.lock:
        s = dg.solver(0)
        stream = dg.stream()
        rnd, done = c_int64(0), c_int(0)
        N.check(L.dawn_sssp_begin(s, int(source), N.GOVM, 0, stream))
        N.check(L.dawn_sssp_advance(s, 1, byref(rnd), byref(done), stream))
        dist = np.empty(n, dtype=np.float64)
        stamp = np.empty(n, dtype=np.uint32)
        N.check(L.dawn_solver_state(s, dist.ctypes.data, stamp.ctypes.data, stream))
        st = N.Stats()
        N.check(L.dawn_solver_result(s, None, None, byref(st), stream))
    # The device round gives the seeded values; the reference's write
    # sequence (which duplicate source->j edge "writes", solver.py:231-249)
    # is the row in CSR order, replayed over its deg(source) edges so
    # writes / first_discoveries / write_counts / pred match it exactly.
    lo, hi = int(g.row_ptr[source]), int(g.row_ptr[source + 1])
    cur = {}
    for k in range(lo, hi):
        j = int(g.col[k])
        if j == source:
            continue
        cand = alpha[source] + float(g.val[k])
        before = cur.get(j, alpha[j])
        if before > cand:
            cur[j] = cand
            if write_counts is not None:
                write_counts[j] += 1
            if pred is not None:
                pred[j] = int(source)
            if stats is not None:
                stats.writes += 1
                if before == inf:
                    stats.first_discoveries += 1
    for j in np.flatnonzero(stamp == 1).tolist():
        alpha[j] = float(dist[j])
        delta[j] = True
    if stats is not None:
        stats.relaxations += int(st.relaxations)
        if st.negative_cycle:
            stats.negative_cycle = True
    return alpha, delta


SOLVERS = {"gsvm": gsvm_sssp, "govm": govm_sssp}


# ---------------------------------------------------------------------------
# multi-source drivers
# ---------------------------------------------------------------------------
_ROW_BYTES_BUDGET = 1 << 30  # float64 rows copied back per dawn_mssp call


def _mssp_run(g, sources: list[int], algo: int, device: int, precision: str | None, schedule: str | None,
              rows: np.ndarray, stats, claim: Callable[[], tuple[int, int] | None]) -> None:
    """Solve the source ranges ``claim()`` hands out on one device, writing
    rows ``[lo, hi)`` of ``rows`` (host float64) and ``stats``."""
    dg = device_graph(g, device=device, precision=precision)
    flags = _neg_flags(dg) | _schedule_flag(schedule)
    with dg.lock:
        s = dg.solver(flags)
        while True:
            rng = claim()
            if rng is None:
                return
            lo, hi = rng
            part = np.asarray(sources[lo:hi], dtype=np.int64)
            out = rows[lo:hi].ctypes.data if rows is not None else None  # None: counters only
            N.check(N.lib().dawn_mssp(s, part.ctypes.data, hi - lo, algo, flags, out,
                                      ctypes.addressof(stats) + lo * ctypes.sizeof(N.Stats), dg.stream()))


def _devices_for(workers: int) -> list[int]:
    ndev = N.device_count()
    if ndev < 1:
        N.require_gpu()
    return list(range(min(max(workers, 1), ndev)))


def mssp(g, sources: Sequence[int], algo: str = "govm", workers: int = 1, *,
         precision: str | None = None, schedule: str | None = None) -> list[tuple[DistanceVector, SolveStats]]:
    """Independent solves from each source, results in the given order (solver.py:426-457).

    ``workers`` is the number of GPUs the sources are spread over (capped at
    the visible device count); results are bit-identical for any value.  With
    several GPUs, one host thread per device claims source chunks from a
    shared cursor (the reference's pool hands out chunks dynamically too,
    solver.py:453-457): per-source cost varies by orders of magnitude, so a
    static split would leave devices idle.  ``schedule`` as in
    :func:`gsvm_sssp` (``async``: same rows, per-source counters
    timing-dependent).
    """
    rows, stats = _mssp_core(g, sources, algo, workers, precision, schedule, with_rows=True)
    return [(DistanceVector(dist=rows[i], source=src), _stats_from_native(stats[i]))
            for i, src in enumerate(int(x) for x in sources)]


def mssp_stats(g, sources: Sequence[int], algo: str = "govm", workers: int = 1, *,
               precision: str | None = None, schedule: str | None = None) -> list[SolveStats]:
    """The ``SolveStats`` half of :func:`mssp` only: the device solves every
    source with the same kernels and counters, but no distance row is
    decoded or copied to the host (k x n x 8 bytes saved).  Consumers that
    only aggregate work counters (the μ experiment, benchmarks) use it."""
    _, stats = _mssp_core(g, sources, algo, workers, precision, schedule, with_rows=False)
    return [_stats_from_native(st) for st in stats]


def _mssp_core(g, sources, algo: str, workers: int, precision, schedule, with_rows: bool):
    _schedule_flag(schedule)  # validate before any work
    name = _normalize_algo(algo)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    sources = [int(s) for s in sources]
    for s in sources:
        _check_source(g, s)
    if not sources:
        return None, []
    algo_id = _ALGO[name]
    devs = _devices_for(workers)
    k, n = len(sources), int(g.n)
    rows = _host_array((k, n)) if with_rows else None
    stats = (N.Stats * k)()
    # a claim is bounded by the host rows it writes; without rows, by 1024 sources
    row_cap = max(1, _ROW_BYTES_BUDGET // (8 * max(n, 1))) if with_rows else 1024
    if len(devs) == 1 or k == 1:
        chunk = row_cap
    else:
        # ~8 claims per device, whole 32-source batches of the batched kernel
        chunk = min(row_cap, max(32, -(-k // (8 * len(devs)) // 32) * 32))
    cursor = [0]
    lock = threading.Lock()

    def claim():
        with lock:
            lo = cursor[0]
            if lo >= k:
                return None
            cursor[0] = min(k, lo + chunk)
            return lo, cursor[0]

    if len(devs) == 1 or k == 1:
        _mssp_run(g, sources, algo_id, devs[0], precision, schedule, rows, stats, claim)
    else:
        with ThreadPoolExecutor(max_workers=len(devs)) as ex:
            for f in [ex.submit(_mssp_run, g, sources, algo_id, d, precision, schedule, rows, stats, claim)
                      for d in devs]:
                f.result()
    return rows, stats


def apsp(g, algo: str = "govm", workers: int = 1, sink: Callable[[DistanceVector], None] | None = None, *,
         precision: str | None = None, schedule: str | None = None) -> AggregateStats:
    """Every source in ascending order, rows streamed to ``sink`` (solver.py:460-495).

    Rows are produced in device batches and handed to ``sink`` strictly in
    source order; the n x n matrix is never held.  A sink exception aborts.
    On one GPU the row path is pipelined: the device solves
    tile i+1 (batched kernel, float64 rows into pinned host memory) while a
    consumer thread hands tile i's rows to ``sink``; two pinned buffers
    alternate.
    """
    name = _normalize_algo(algo)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    _schedule_flag(schedule)
    agg = AggregateStats()
    n = g.n
    if n == 0:
        return agg.finish()
    batch = max(1, min(n, (256 << 20) // (8 * n)))
    if workers > 1 and N.device_count() > 1:
        for lo in range(0, n, batch):
            for dv, st in mssp(g, range(lo, min(n, lo + batch)), name, workers, precision=precision,
                               schedule=schedule):
                if sink is not None:
                    sink(dv)
                agg.add(st)
        return agg.finish()
    return _apsp_pipelined(g, name, sink, precision, batch, agg, schedule)


def _apsp_pipelined(g, name: str, sink, precision, batch: int, agg: AggregateStats,
                    schedule: str | None = None) -> AggregateStats:
    import queue

    import torch

    dg = device_graph(g, precision=precision)
    n = dg.n
    algo_id = _ALGO[name]
    flags = _neg_flags(dg) | _schedule_flag(schedule)
    bufs = [torch.empty((batch, n), dtype=torch.float64).pin_memory() for _ in range(2)]
    free: "queue.Queue[int]" = queue.Queue()
    for i in range(2):
        free.put(i)
    ready: "queue.Queue" = queue.Queue()
    failure: list[BaseException] = []

    def consume():
        while True:
            item = ready.get()
            if item is None:
                return
            slot, lo, k, stats = item
            try:
                if not failure:
                    rows = np.array(bufs[slot][:k].numpy())  # fresh arrays: the buffer is reused
                    for i in range(k):
                        if sink is not None:
                            sink(DistanceVector(dist=rows[i], source=lo + i))
                        agg.add(_stats_from_native(stats[i]))
            except BaseException as e:  # a sink exception aborts apsp (solver.py:470-471)
                failure.append(e)
            finally:
                free.put(slot)

    worker = threading.Thread(target=consume, daemon=True)
    worker.start()
    try:
        with dg.lock:
            s = dg.solver(flags)
            for lo in range(0, n, batch):
                slot = free.get()
                if failure:
                    break
                k = min(batch, n - lo)
                srcs = np.arange(lo, lo + k, dtype=np.int64)
                stats = (N.Stats * k)()
                N.check(N.lib().dawn_mssp(s, srcs.ctypes.data, k, algo_id, flags, bufs[slot].data_ptr(),
                                          ctypes.addressof(stats), dg.stream()))
                ready.put((slot, lo, k, stats))
    finally:
        ready.put(None)
        worker.join()
    if failure:
        raise failure[0]
    return agg.finish()


def format_distance_row(dv: DistanceVector) -> str:
    """``source,d0,d1,...`` with ``%.17g`` and the literal ``inf`` (solver.py:498-506).

    Long rows go through the native multi-threaded formatter
    (``dawn_format_rows``, same text byte for byte)."""
    dist = np.asarray(dv.dist, dtype=np.float64)
    if dist.size >= 2048:
        return format_distance_rows(dist[None, :], [dv.source])[:-1]
    return ",".join([str(dv.source)] + ["inf" if d == inf else "%.17g" % d for d in dist.tolist()])


def format_distance_rows(rows, sources, threads: int = 0) -> str:
    """Rows ``[k][n]`` (float64, any row stride) as ``k`` lines of
    :func:`format_distance_row` text, each ending in a newline (SURVEY §8(f)
    F2: the APSP text output path, ~20-40x the Python loop on 16 threads)."""
    rows = np.asarray(rows, dtype=np.float64)
    if rows.ndim != 2 or rows.strides[1] != 8:
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(len(sources), -1)
    k, n = rows.shape
    src = np.ascontiguousarray([int(x) for x in sources], dtype=np.int64)
    if src.size != k:
        raise ValueError("one source per row")
    cap = k * (24 + 26 * n)
    buf = ctypes.create_string_buffer(max(cap, 1))
    ln = ctypes.c_int64(0)
    ld = rows.strides[0] // 8 if k > 1 else n  # a single row may carry a 0 stride (x[None, :])
    N.check(N.lib().dawn_format_rows(rows.ctypes.data, k, n, ld, src.ctypes.data, buf, cap, byref(ln),
                                     int(threads)))
    return buf.raw[: ln.value].decode("ascii")


_ROWS_MAGIC = b"DAWNROWS"


def write_distance_rows(fh, rows, sources, fmt: str = "text") -> int:
    """Stream rows to a file object: ``text`` = :func:`format_distance_rows`
    lines; ``binary`` = ``b"DAWNROWS"``, int64 k, int64 n, int64 sources[k],
    float64 rows[k][n] little-endian (no formatting cost, exact values).
    Returns the bytes written."""
    rows = np.asarray(rows, dtype=np.float64)
    if fmt == "text":
        data = format_distance_rows(rows, sources).encode("ascii")
        fh.write(data)
        return len(data)
    if fmt != "binary":
        raise ValueError(f"unknown row format {fmt!r}; expected 'text' or 'binary'")
    k, n = rows.shape
    src = np.ascontiguousarray([int(x) for x in sources], dtype="<i8")
    parts = [_ROWS_MAGIC, np.array([k, n], dtype="<i8").tobytes(), src.tobytes(),
             np.ascontiguousarray(rows, dtype="<f8").tobytes()]
    for p_ in parts:
        fh.write(p_)
    return sum(len(p_) for p_ in parts)


def read_distance_rows(fh) -> tuple[np.ndarray, np.ndarray]:
    """Inverse of ``write_distance_rows(..., fmt="binary")``: (sources, rows)."""
    if fh.read(8) != _ROWS_MAGIC:
        raise ValueError("not a DAWNROWS stream")
    k, n = np.frombuffer(fh.read(16), dtype="<i8").tolist()
    src = np.frombuffer(fh.read(8 * k), dtype="<i8").copy()
    rows = np.frombuffer(fh.read(8 * k * n), dtype="<f8").reshape(k, n).copy()
    return src, rows
