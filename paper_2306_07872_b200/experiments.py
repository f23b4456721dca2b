"""The paper's μ experiment on the device.

API of the reference's ``run_mu_experiment`` / ``MuReport``
(``sparsepath/experiments.py:55-92``, ``:127-178``): same arguments, source
sample, weight arms, error texts and report layout, so the reference's
callers and tests take this module unchanged.

The work is organised differently.  The experiment only consumes work
counters, so each arm is one counters-only multi-source run
(:func:`solver.mssp_stats`): the batched kernel advances 32 sources per pass
and no distance row is decoded or copied back (the reference materialises
every row in Python).  The two arms share one structure; each is uploaded once
and cached by the device-graph cache.

Counters follow the device's snapshot-Jacobi rounds.  The
unit-weight arm equals the reference's exactly (every path is discovered once
in either order: μ = 1, no re-updates).  The randomized arm's μ and updated
ratio are the Jacobi figures: deterministic, not the reference's Gauss–Seidel
counts on large graphs.
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np

from .graph import WeightMode, apply_weight_mode
from .solver import AggregateStats, aggregate_stats, mssp_stats

__all__ = ["MuReport", "run_mu_experiment", "RANDOM_WEIGHT_LO", "RANDOM_WEIGHT_HI"]

# the randomized arm draws U[lo, hi) weights (experiments.py:51-52)
RANDOM_WEIGHT_LO = 0.0
RANDOM_WEIGHT_HI = 2.0


@dataclass
class MuReport:
    """Unit-weight arm vs random-weight arm over one structure (experiments.py:55-92).

    Field order is the serialisation order of :meth:`to_dict` /
    :meth:`to_flat_dict`; the two ``AggregateStats`` fields serialise as their
    ``as_dict()`` (nested) or as ``<arm>_<key>`` columns (flat)."""

    graph_id: str
    sources_sampled: int
    baseline: AggregateStats
    randomized: AggregateStats
    mean_updated_ratio: float
    mean_mu: float
    seed: int
    notes: str = ""

    def _items(self):
        for f in fields(self):
            yield f.name, getattr(self, f.name)

    def to_dict(self) -> dict:
        return {k: (v.as_dict() if isinstance(v, AggregateStats) else v) for k, v in self._items()}

    def to_flat_dict(self) -> dict:
        out: dict = {}
        for k, v in self._items():
            if isinstance(v, AggregateStats):
                out.update((f"{k}_{sub}", x) for sub, x in v.as_dict().items())
            else:
                out[k] = v
        return out


def _sample(n: int, wanted: int, seed: int) -> tuple[list[int], str]:
    """The seeded source sample (experiments.py:141-155): ``wanted`` distinct
    nodes, ascending, clamped to ``n`` with a note."""
    if wanted < 1:
        raise ValueError("num_sources must be >= 1")
    if n == 0:
        raise ValueError("cannot sample sources from an empty graph")
    note = ""
    if wanted > n:
        note, wanted = f"requested {wanted} sources, clamped to n={n}", n
    picked = np.random.default_rng(seed).choice(n, size=wanted, replace=False)
    return sorted(map(int, picked)), note


def _arm(g, mode: WeightMode, sources: list[int], workers: int) -> AggregateStats:
    """One arm: ``g``'s structure under ``mode``, counters only, on the device."""
    return aggregate_stats(mssp_stats(apply_weight_mode(g, mode), sources, "govm", workers))


def run_mu_experiment(g, num_sources: int = 64, seed: int = 0, workers: int = 1,
                      graph_id: str | None = None) -> MuReport:
    """Unit weights vs U[0, 2) weights from the same seeded sources
    (experiments.py:127-178).  ``seed`` drives both the sample and the random
    weights, so reports are identical across runs and ``workers`` (GPUs)."""
    sources, note = _sample(g.n, num_sources, seed)
    unit = _arm(g, WeightMode.unit(), sources, workers)
    if unit.re_updates:
        # unit weights reach every node along its fewest-hop path in one write
        raise RuntimeError(
            "unit-weight baseline produced re-updates; the frontier kernel "
            "is expected to discover each path exactly once"
        )
    rand = _arm(g, WeightMode.random_uniform(RANDOM_WEIGHT_LO, RANDOM_WEIGHT_HI, seed=seed), sources, workers)
    return MuReport(
        graph_id=graph_id if graph_id is not None else f"graph(n={g.n},m={g.m})",
        sources_sampled=len(sources),
        baseline=unit,
        randomized=rand,
        mean_updated_ratio=rand.mean_updated_ratio,
        mean_mu=rand.mean_mu,
        seed=seed,
        notes=note,
    )
