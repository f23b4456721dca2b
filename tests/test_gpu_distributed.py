"""The multi-rank APSP driver's CUDA path on one GPU: two processes (gloo for
control) share cuda:0, rank 1's rows reach rank 0's tile through CUDA IPC +
copy-engine peer copies (transport "p2p") — the same code the 8-GPU run uses,
with both ranks on one device."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph():
    from paper_2306_07872_b200 import generators as G

    return G.rmat_graph(12, 8, weights="f32")


def _sources(n):
    rng = np.random.default_rng(7)
    return [int(x) for x in rng.integers(0, n, 101)]


def _worker(rank, world, port, out_dir, transport):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2306_07872_b200 import multisource as MS

    g = _graph()
    src = _sources(g.n)
    res = MS.apsp_sharded(g, src, "govm", precision="fp32", transport=transport)
    assert res.transport == transport
    if rank == 0:
        np.save(os.path.join(out_dir, "tile.npy"), res.tile.cpu().numpy())
        np.save(os.path.join(out_dir, "steps.npy"), np.array([s.relaxations for s in res.stats]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["p2p"])
def test_apsp_sharded_two_ranks_one_gpu(gpu, tmp_path, transport):
    from paper_2306_07872_b200 import multisource as MS

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), transport), nprocs=2, join=True)
    tile = np.load(tmp_path / "tile.npy")
    relax = np.load(tmp_path / "steps.npy")
    g = _graph()
    src = _sources(g.n)
    ref, stats = MS.mssp_tile(g, src, "govm", precision="fp32")
    import torch

    assert tile.dtype == np.float32
    assert np.array_equal(tile.astype(np.float64), ref.cpu().numpy())
    assert relax.tolist() == [s.relaxations for s in stats]
