"""Device-resident graphs and solvers (the upload side of the C ABI).

A ``CsrGraph`` is uploaded once per (graph object, device, precision) and
cached by object identity — the reference's ``CsrGraph`` is frozen and
identity-hashed (graph.py:64), so a cache hit is always the same arrays.
The reference instead re-converts the CSR with ``.tolist()`` on every solve
(solver.py:272-274, :340-342).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from ctypes import byref, c_int, c_int64, c_void_p

import numpy as np

from . import _native as N

_cache_lock = threading.Lock()
_cache: "weakref.WeakKeyDictionary[object, dict]" = weakref.WeakKeyDictionary()
_strong_cache: dict[int, tuple[object, dict]] = {}

_default_precision = "auto"
_default_schedule = "jacobi"
_tuning: dict[str, float] = {}
SCHEDULES = ("jacobi", "async")


def set_tuning(**knobs: float) -> None:
    """Process-wide solver tuning (``dawn_solver_tune``); results never depend on it.

    ``dense_edges_per_node``: rounds relaxing >= value * n edges rebuild the
    next frontier by a coalesced sweep instead of an enqueue (default 0.5).
    Applies to solvers created afterwards and to existing cached ones.
    """
    _tuning.update({k: float(v) for k, v in knobs.items()})
    with _cache_lock:
        for per in list(_cache.values()):
            for dg in per.values():
                dg.retune()
        for _, per in _strong_cache.values():
            for dg in per.values():
                dg.retune()


def set_default_precision(precision: str) -> None:
    """Process-wide precision policy: ``auto`` (exact: integer weights on the
    integer path, everything else float64), ``fp32`` (opt-in, <=1e-6 relative)
    or ``fp64``."""
    global _default_precision
    if precision not in N.PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}; expected one of {sorted(N.PRECISIONS)}")
    _default_precision = precision


def get_default_precision() -> str:
    return _default_precision


def set_default_schedule(schedule: str) -> None:
    """Process-wide round schedule of the single-source solvers.

    ``jacobi`` (default): every frontier row is relaxed with its value at the
    start of the round — distances AND work counters are deterministic and
    equal to the snapshot-Jacobi oracle.  ``async``: rows are relaxed with
    their live value, which another row may already have lowered in the same
    round (the reference's in-place order, solver.py:369-385, does the same
    sequentially): identical distances and negative-cycle flags, fewer
    relaxations (C2: 212 M instead of 299 M), counters timing-dependent.
    """
    global _default_schedule
    if schedule not in SCHEDULES:
        raise ValueError(f"unknown schedule {schedule!r}; expected one of {list(SCHEDULES)}")
    _default_schedule = schedule


def get_default_schedule() -> str:
    return _default_schedule


def _current_stream(device: int) -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return int(torch.cuda.current_stream(device).cuda_stream)
    except Exception:  # torch missing or no CUDA: the legacy default stream
        pass
    return 0


def _default_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return int(torch.cuda.current_device())
    except Exception:
        pass
    return 0


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class DeviceGraph:
    """One graph resident in HBM plus its per-flag solvers."""

    def __init__(self, handle: int, device: int, n: int, m: int, vtype: int):
        self.handle = handle
        self.device = device
        self.n = n
        self.m = m
        self.vtype = vtype
        self._solvers: dict[int, int] = {}
        self.lock = threading.RLock()

    # -- construction -------------------------------------------------------
    @classmethod
    def from_csr(cls, g, device: int | None = None, precision: str | None = None) -> "DeviceGraph":
        N.require_gpu()
        device = _default_device() if device is None else device
        prec = N.PRECISIONS[precision or _default_precision]
        rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(g.col, dtype=np.int64)
        val = np.ascontiguousarray(g.val, dtype=np.float64)
        vt = c_int(0)
        N.check(N.lib().dawn_choose_vtype(int(g.n), int(g.m), _ptr(val) if g.m else None, prec, byref(vt)))
        h = c_void_p()
        N.check(N.lib().dawn_graph_create(device, int(g.n), int(g.m), _ptr(rp), _ptr(col) if g.m else None,
                                          _ptr(val) if g.m else None, vt.value, 0, byref(h)))
        return cls(h.value, device, int(g.n), int(g.m), vt.value)

    @classmethod
    def from_device_arrays(cls, n: int, m: int, row_ptr, col, val, vtype: int, device: int) -> "DeviceGraph":
        """Upload from device tensors (int64 row_ptr/col, float64 val) without a host round trip."""
        N.require_gpu()
        h = c_void_p()
        N.check(N.lib().dawn_graph_create(device, int(n), int(m), row_ptr.data_ptr(), col.data_ptr(),
                                          val.data_ptr(), int(vtype), 1, byref(h)))
        return cls(h.value, device, int(n), int(m), int(vtype))

    # -- solvers ------------------------------------------------------------
    def solver(self, flags: int = 0) -> int:
        key = flags & (N.F_PRED | N.F_NEGCHECK | N.F_PROFILE)
        with self.lock:
            s = self._solvers.get(key)
            if s is None:
                h = c_void_p()
                N.check(N.lib().dawn_solver_create(self.handle, key, byref(h)))
                s = self._solvers[key] = h.value
                self._apply_tuning(s)
            return s

    def _apply_tuning(self, s: int) -> None:
        for k, v in _tuning.items():
            N.check(N.lib().dawn_solver_tune(s, k.encode(), v))

    def retune(self) -> None:
        with self.lock:
            for s in self._solvers.values():
                self._apply_tuning(s)

    def device_bytes(self) -> int:
        b = c_int64(0)
        N.check(N.lib().dawn_graph_info(self.handle, None, None, None, byref(b)))
        return b.value

    def stream(self) -> int:
        return _current_stream(self.device)

    @property
    def vtype_name(self) -> str:
        return N.VTYPE_NAMES[self.vtype]

    def close(self) -> None:
        L = N._lib
        if L is None or self.handle is None:
            return
        for s in self._solvers.values():
            L.dawn_solver_destroy(s)
        self._solvers.clear()
        L.dawn_graph_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_graph(g, device: int | None = None, precision: str | None = None) -> DeviceGraph:
    """Cached upload of ``g`` (see module doc)."""
    if isinstance(g, DeviceGraph):
        return g
    device = _default_device() if device is None else device
    key = (device, precision or _default_precision)
    with _cache_lock:
        try:
            per = _cache.get(g)
            if per is None:
                per = {}
                _cache[g] = per
        except TypeError:  # not weak-referenceable: keep it alive with the upload
            ent = _strong_cache.get(id(g))
            if ent is None or ent[0] is not g:
                ent = (g, {})
                _strong_cache[id(g)] = ent
            per = ent[1]
        dg = per.get(key)
        if dg is None:
            dg = DeviceGraph.from_csr(g, device=device, precision=key[1])
            per[key] = dg
        return dg


def clear_cache() -> None:
    with _cache_lock:
        for per in list(_cache.values()):
            for dg in per.values():
                dg.close()
        _cache.clear()
        for _, per in _strong_cache.values():
            for dg in per.values():
                dg.close()
        _strong_cache.clear()
