"""Device-side synthetic graph construction for large configurations.

``dawn_gen_rmat`` (csrc/dawn.cu) draws the RMAT edge list on the GPU with the
same counter hash as :mod:`generators` (so the graph is bit-identical to the
host restatement), then the canonical CSR order — rows by source, columns
ascending, ties in generation order (reference graph.py:303-322) — comes from
a stable device sort of the 64-bit key ``u*n + v``.  torch supplies the sort
and buffers here (plumbing); the graph is handed to ``dawn_graph_create``
without a host round trip.
"""

from __future__ import annotations

from . import _native as N
from .device import DeviceGraph
from .graph import CsrGraph


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
    key = u * n + v
    _, order = torch.sort(key, stable=True)
    del key
    col = v[order]
    val = w[order]
    counts = torch.bincount(u, minlength=n)
    del u, v, w, order
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=row_ptr[1:])
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
