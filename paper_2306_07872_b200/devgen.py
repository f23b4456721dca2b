"""Device-side graph construction.

``dawn_gen_rmat`` (csrc/dawn.cu) draws the RMAT edge list on the GPU with the
same counter hash as :mod:`generators` (so the graph is bit-identical to the
host restatement); ``dawn_build_csr`` (csrc/dawn_csr.cuh) then puts any edge
list in the canonical CSR order of the reference's ``build_csr`` — rows by
source, columns ascending, ties in input order (graph.py:303-322) — with a
stable device radix sort of the 64-bit key ``u*n + v``.  torch only holds
the buffers; the graph reaches ``dawn_graph_create`` without a host round trip.
"""

from __future__ import annotations

from . import _native as N
from .device import DeviceGraph
from .graph import CsrGraph


def csr_device(n: int, u, v, w, device: int = 0):
    """Canonical CSR (reference build_csr order, graph.py:303-322) built on the
    device by ``dawn_build_csr``: int64 ``row_ptr[n+1]``, int64 ``col[m]``,
    float64 ``val[m]`` CUDA tensors.  ``u``/``v``/``w`` are CUDA tensors or
    host arrays (int64, int64, float64)."""
    import numpy as np
    import torch

    dev = torch.device("cuda", device)
    on_dev = isinstance(u, torch.Tensor) and u.is_cuda
    if on_dev:
        u = u.to(torch.int64).contiguous()
        v = v.to(torch.int64).contiguous()
        w = w.to(torch.float64).contiguous()
        m = int(u.numel())
        pu, pv, pw = u.data_ptr(), v.data_ptr(), w.data_ptr()
    else:
        u = np.ascontiguousarray(u, dtype=np.int64)
        v = np.ascontiguousarray(v, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        m = int(u.size)
        pu, pv, pw = (u.ctypes.data, v.ctypes.data, w.ctypes.data) if m else (None, None, None)
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    val = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(N.lib().dawn_build_csr(device, n, m, pu, pv, pw, 1 if on_dev else 0, row_ptr.data_ptr(),
                                   col.data_ptr(), val.data_ptr(), stream))
    return row_ptr, col[:m], val[:m]


def build_csr_device(n: int, u, v, w, device: int = 0) -> CsrGraph:
    """``build_csr`` on the GPU, returned as the reference's host ``CsrGraph``."""
    rp, col, val = csr_device(n, u, v, w, device=device)
    return CsrGraph(n=n, m=int(col.numel()), row_ptr=rp.cpu().numpy(), col=col.cpu().numpy(),
                    val=val.cpu().numpy())


def rmat_csr_device(scale: int, edge_factor: int, weights: str = "f32", lo: int = 1, hi: int = 100, seed: int = 1,
                    wseed: int = 2, device: int = 0, a: float = 0.57, b: float = 0.19, c: float = 0.19):
    """Return (n, m, row_ptr, col, val) torch CUDA tensors (int64, int64, float64)."""
    import torch

    n = 1 << scale
    m = edge_factor * n
    dev = torch.device("cuda", device)
    u = torch.empty(m, dtype=torch.int64, device=dev)
    v = torch.empty(m, dtype=torch.int64, device=dev)
    w = torch.empty(m, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(N.lib().dawn_gen_rmat(device, scale, edge_factor, a, b, c, seed, 0 if weights == "int" else 1, lo, hi,
                                  wseed, u.data_ptr(), v.data_ptr(), w.data_ptr(), stream))
    row_ptr, col, val = csr_device(n, u, v, w, device=device)
    del u, v, w
    return n, m, row_ptr, col, val


def rmat_device_graph(scale: int, edge_factor: int, weights: str = "f32", precision: str = "fp32",
                      device: int = 0, keep_host: bool = False, **kw):
    """Build an RMAT graph directly in HBM; optionally also return the host
    ``CsrGraph`` (for the oracle / CPU baseline / end-to-end API path)."""
    import numpy as np

    n, m, rp, col, val = rmat_csr_device(scale, edge_factor, weights=weights, device=device, **kw)
    vt = {"fp32": N.F32, "fp64": N.F64}.get(precision)
    if vt is None:  # auto: integer weights -> int32 when the bound allows
        import ctypes

        hv = val.cpu().numpy()
        c = ctypes.c_int(0)
        N.check(N.lib().dawn_choose_vtype(n, m, hv.ctypes.data, N.PREC_AUTO, ctypes.byref(c)))
        vt = c.value
    dg = DeviceGraph.from_device_arrays(n, m, rp, col, val, vt, device)
    host = None
    if keep_host:
        host = CsrGraph(n=n, m=m, row_ptr=rp.cpu().numpy(), col=col.cpu().numpy(), val=val.cpu().numpy())
    deg = (rp[1:] - rp[:-1]).clone()
    del rp, col, val
    return dg, host, deg


def grid_csr_device(rows: int, cols: int, weights: str = "int", lo: int = 1, hi: int = 100, wseed: int = 2,
                    device: int = 0):
    """``grid_graph`` (generators.py) written straight into CSR on the device
    by ``dawn_gen_grid``: (n, m, row_ptr, col, val) CUDA tensors."""
    import torch

    n = rows * cols
    m = 4 * rows * cols - 2 * rows - 2 * cols
    dev = torch.device("cuda", device)
    rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    val = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(N.lib().dawn_gen_grid(device, rows, cols, 0 if weights == "int" else 1, lo, hi, wseed, rp.data_ptr(),
                                  col.data_ptr(), val.data_ptr(), stream))
    return n, m, rp, col[:m], val[:m]


def grid_device_graph(rows: int, cols: int, precision: str = "fp32", device: int = 0, keep_host: bool = False,
                      **kw):
    """A resident ``DeviceGraph`` of the grid (no host build, no sort);
    optionally also the host ``CsrGraph``."""
    n, m, rp, col, val = grid_csr_device(rows, cols, device=device, **kw)
    vt = {"fp32": N.F32, "fp64": N.F64, "int32": N.I32}[precision]
    dg = DeviceGraph.from_device_arrays(n, m, rp, col, val, vt, device)
    host = None
    if keep_host:
        host = CsrGraph(n=n, m=m, row_ptr=rp.cpu().numpy(), col=col.cpu().numpy(), val=val.cpu().numpy())
    return dg, host
