"""The paper's μ experiment on the GPU.

Mirror of ``run_mu_experiment`` / ``MuReport`` (reference experiments.py:55-92,
:127-178): the same seeded source sample, the same unit-weight baseline and
U[0, 2) randomized arm over one graph structure, the same checks and report
fields.  Both arms run through :func:`mssp`, i.e. the batched multi-source
kernel (32 sources per pass) — the reference solves one source at a time in
Python.

Counters follow the device's snapshot-Jacobi rounds: the
baseline arm is identical to the reference's (unit weights discover every
path exactly once, so μ = 1 and re_updates = 0 in both orders); the
randomized arm's μ and updated ratio are the Jacobi figures, deterministic but
not equal to the reference's Gauss-Seidel counts on large graphs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .graph import WeightMode, apply_weight_mode
from .solver import AggregateStats, aggregate_stats, mssp

__all__ = ["MuReport", "run_mu_experiment", "RANDOM_WEIGHT_LO", "RANDOM_WEIGHT_HI"]

RANDOM_WEIGHT_LO = 0.0  # reference experiments.py:51-52
RANDOM_WEIGHT_HI = 2.0


@dataclass
class MuReport:
    """Paired unit-weight vs random-weight statistics for one graph (experiments.py:55-92)."""

    graph_id: str
    sources_sampled: int
    baseline: AggregateStats
    randomized: AggregateStats
    mean_updated_ratio: float
    mean_mu: float
    seed: int
    notes: str = ""

    def to_dict(self) -> dict:
        return {
            "graph_id": self.graph_id,
            "sources_sampled": self.sources_sampled,
            "baseline": self.baseline.as_dict(),
            "randomized": self.randomized.as_dict(),
            "mean_updated_ratio": self.mean_updated_ratio,
            "mean_mu": self.mean_mu,
            "seed": self.seed,
            "notes": self.notes,
        }

    def to_flat_dict(self) -> dict:
        flat: dict = {"graph_id": self.graph_id, "sources_sampled": self.sources_sampled}
        for prefix, agg in (("baseline", self.baseline), ("randomized", self.randomized)):
            for key, value in agg.as_dict().items():
                flat[f"{prefix}_{key}"] = value
        flat["mean_updated_ratio"] = self.mean_updated_ratio
        flat["mean_mu"] = self.mean_mu
        flat["seed"] = self.seed
        flat["notes"] = self.notes
        return flat


def run_mu_experiment(g, num_sources: int = 64, seed: int = 0, workers: int = 1,
                      graph_id: str | None = None) -> MuReport:
    """Unit-weight baseline vs U[0, 2) weights from a seeded source sample
    (reference experiments.py:127-178: same arguments, validation, sampling and
    errors)."""
    if num_sources < 1:
        raise ValueError("num_sources must be >= 1")
    if g.n == 0:
        raise ValueError("cannot sample sources from an empty graph")
    notes = ""
    if num_sources > g.n:
        notes = f"requested {num_sources} sources, clamped to n={g.n}"
        num_sources = g.n
    if graph_id is None:
        graph_id = f"graph(n={g.n},m={g.m})"

    rng = np.random.default_rng(seed)
    sources = sorted(int(s) for s in rng.choice(g.n, size=num_sources, replace=False))

    unit = apply_weight_mode(g, WeightMode.unit())
    randomized = apply_weight_mode(g, WeightMode.random_uniform(RANDOM_WEIGHT_LO, RANDOM_WEIGHT_HI, seed=seed))

    base_agg = aggregate_stats(s for _, s in mssp(unit, sources, "govm", workers))
    if base_agg.re_updates != 0:
        raise RuntimeError(
            "unit-weight baseline produced re-updates; the frontier kernel "
            "is expected to discover each path exactly once"
        )
    rand_agg = aggregate_stats(s for _, s in mssp(randomized, sources, "govm", workers))
    return MuReport(
        graph_id=graph_id,
        sources_sampled=num_sources,
        baseline=base_agg,
        randomized=rand_agg,
        mean_updated_ratio=rand_agg.mean_updated_ratio,
        mean_mu=rand_agg.mean_mu,
        seed=seed,
        notes=notes,
    )
