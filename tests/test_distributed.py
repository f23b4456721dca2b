"""Multi-rank source sharding on CPU: world_size 2 and 3 over
gloo.  The device solve is replaced by the oracle (``solve_fn``) so the host
logic — dynamic batch claiming from the group-wide cursor, point-to-point
delivery into the root tile in source order, the stats all-reduce, the load
all-gather, max-over-ranks timing — runs without a GPU."""

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


def _worker(rank, world, port, sources, out_dir, claim="dynamic"):
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

    res = MS.apsp_sharded(g, sources, "govm", solve_fn=solve_fn, out_dtype=torch.float64, claim=claim)
    assert res.transport == "collective"
    bounds = MS.batch_bounds(len(sources))
    assert [tuple(x) for x in solved] == [bounds[b] for b in res.claimed]
    if claim == "static":
        assert [tuple(x) for x in solved] == MS.shard_batches(len(sources), world)[rank]
    # every rank holds every source's counters after the all-reduce
    lines = [f"{st.outer_steps} {st.relaxations} {st.writes} {st.first_discoveries} {st.updated_ratio!r}"
             for st in res.stats]
    with open(os.path.join(out_dir, f"stats{rank}.txt"), "w") as f:
        f.write("\n".join(lines))
    with open(os.path.join(out_dir, f"claimed{rank}.txt"), "w") as f:
        f.write(" ".join(map(str, res.claimed)))
    assert sorted(p["rank"] for p in res.per_rank) == list(range(world))
    assert sum(p["batches"] for p in res.per_rank) == len(bounds)
    if rank == 0:
        np.save(os.path.join(out_dir, "tile.npy"), res.tile.numpy())
    else:
        assert res.tile is None
    dist.destroy_process_group()


@pytest.mark.parametrize("world,claim", [(2, "dynamic"), (3, "dynamic"), (2, "static")])
def test_apsp_sharded_gloo(tmp_path, world, claim):
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    sources = [int(x) for x in rng.integers(0, 90, 101)]  # 4 batches: uneven deal
    mp.spawn(_worker, args=(world, _free_port(), sources, str(tmp_path), claim), nprocs=world, join=True)
    tile = np.load(tmp_path / "tile.npy")
    g = _graph()
    assert tile.shape == (len(sources), g.n)
    claimed = sorted(int(b) for r in range(world) for b in (tmp_path / f"claimed{r}.txt").read_text().split())
    assert claimed == list(range(4)), "every batch claimed exactly once"
    per_rank = [(tmp_path / f"stats{r}.txt").read_text().split("\n") for r in range(world)]
    assert all(p == per_rank[0] for p in per_rank)
    for i, s in enumerate(sources):
        d, _, o = O.jacobi_sssp(g, s, "govm", vtype="int32")
        assert np.array_equal(tile[i], d)
        assert per_rank[0][i].split()[:4] == [str(o[k]) for k in ("outer_steps", "relaxations", "writes",
                                                                  "first_discoveries")]


def _skew_worker(rank, world, port, out_dir, claim):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    import time

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2306_07872_b200 import multisource as MS
    from paper_2306_07872_b200.solver import SolveStats

    g = _graph()
    sources = [i % g.n for i in range(32 * 12)]  # 12 batches

    def solve_fn(lo, hi):
        time.sleep(0.30 if lo == 0 else 0.05)  # batch 0 holds the expensive sources (hub rows)
        return torch.zeros((hi - lo, g.n), dtype=torch.float64), [SolveStats() for _ in range(hi - lo)]

    res = MS.apsp_sharded(g, sources, "govm", solve_fn=solve_fn, claim=claim)
    if rank == 0:
        import json

        with open(os.path.join(out_dir, f"skew_{claim}.json"), "w") as f:
            json.dump({"per_rank": res.per_rank, "ms_max": res.ms_max}, f)
    dist.destroy_process_group()


def test_dynamic_claiming_balances_skewed_cost(tmp_path):
    """One batch costs 6x the others: the dynamic cursor lets the other rank
    take the cheap batches while the expensive one runs; the static deal
    leaves the expensive batch's rank with half the cheap ones too."""
    import json

    for claim in ("dynamic", "static"):
        mp.spawn(_skew_worker, args=(2, _free_port(), str(tmp_path), claim), nprocs=2, join=True)
    dyn = json.loads((tmp_path / "skew_dynamic.json").read_text())
    sta = json.loads((tmp_path / "skew_static.json").read_text())
    assert [p["batches"] for p in sta["per_rank"]] == [6, 6]
    nb = sorted(p["batches"] for p in dyn["per_rank"])
    assert nb[0] <= 4 and nb[1] >= 8 and sum(nb) == 12, dyn  # ~balanced time, not count
    # makespan: static >= 0.30 + 5 x 0.05 = 0.55 s; balanced dynamic ~0.43 s
    assert sta["ms_max"] >= 540
    assert dyn["ms_max"] < sta["ms_max"] - 60, (dyn, sta)


def test_shard_batches_deal():
    from paper_2306_07872_b200.multisource import shard_batches

    assert shard_batches(0, 4) == [[], [], [], []]
    assert shard_batches(70, 2) == [[(0, 32), (64, 70)], [(32, 64)]]
    deal = shard_batches(8192, 8)
    assert all(len(d) == 32 for d in deal)
    covered = sorted(x for d in deal for x in d)
    assert covered[0][0] == 0 and covered[-1][1] == 8192
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
