"""Multi-rank source sharding on CPU: world_size 2 and 3 over
gloo.  The device solve is replaced by the oracle (``solve_fn``) so the host
logic — round-robin batch deal, point-to-point delivery into the root tile in
source order, stats gathering, max-over-ranks timing — runs without a GPU."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph():
    from paper_2306_07872_b200 import csr_from_arrays

    rng = np.random.default_rng(3)
    n, m = 90, 500
    return csr_from_arrays(n, rng.integers(0, n, m), rng.integers(0, n, m), rng.integers(1, 30, m).astype(float))


def _worker(rank, world, port, sources, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from paper_2306_07872_b200 import multisource as MS
    from paper_2306_07872_b200.solver import SolveStats

    g = _graph()
    solved = []

    def solve_fn(lo, hi):
        rows, sts = [], []
        for s in sources[lo:hi]:
            d, _, o = O.jacobi_sssp(g, s, "govm", vtype="int32")
            rows.append(torch.from_numpy(d))
            sts.append(SolveStats(outer_steps=o["outer_steps"], relaxations=o["relaxations"], writes=o["writes"],
                                  first_discoveries=o["first_discoveries"]))
        solved.append((lo, hi))
        return torch.stack(rows), sts

    res = MS.apsp_sharded(g, sources, "govm", solve_fn=solve_fn, out_dtype=torch.float64)
    assert res.transport == "collective"
    assert [tuple(x) for x in solved] == MS.shard_batches(len(sources), world)[rank]
    if rank == 0:
        np.save(os.path.join(out_dir, "tile.npy"), res.tile.numpy())
        with open(os.path.join(out_dir, "stats.txt"), "w") as f:
            for st in res.stats:
                f.write(f"{st.outer_steps} {st.relaxations} {st.writes} {st.first_discoveries}\n")
    else:
        assert res.tile is None and res.stats is None
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_apsp_sharded_gloo(tmp_path, world):
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    sources = [int(x) for x in rng.integers(0, 90, 101)]  # 4 batches: uneven deal
    mp.spawn(_worker, args=(world, _free_port(), sources, str(tmp_path)), nprocs=world, join=True)
    tile = np.load(tmp_path / "tile.npy")
    lines = (tmp_path / "stats.txt").read_text().split("\n")
    g = _graph()
    assert tile.shape == (len(sources), g.n)
    for i, s in enumerate(sources):
        d, _, o = O.jacobi_sssp(g, s, "govm", vtype="int32")
        assert np.array_equal(tile[i], d)
        assert lines[i] == f"{o['outer_steps']} {o['relaxations']} {o['writes']} {o['first_discoveries']}"


def test_shard_batches_deal():
    from paper_2306_07872_b200.multisource import shard_batches

    assert shard_batches(0, 4) == [[], [], [], []]
    assert shard_batches(70, 2) == [[(0, 32), (64, 70)], [(32, 64)]]
    deal = shard_batches(8192, 8)
    assert all(len(d) == 32 for d in deal)
    covered = sorted(x for d in deal for x in d)
    assert covered[0][0] == 0 and covered[-1][1] == 8192
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
