"""Golden μ-experiment reports from the REFERENCE (run in the build container:
it imports /root/reference/pkg/src).  Writes tests/golden/mu_reports.json.

Cases: the reference's own seeded Erdos-Renyi generator
(graph.py:405-453) at three sizes, run_mu_experiment (experiments.py:127-178)
with 16-64 sources."""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import sparsepath as R  # noqa: E402

CASES = [(200, 4.0, 1, 16, 0), (600, 6.0, 2, 32, 3), (1500, 3.0, 5, 64, 7)]


def main():
    out = []
    for n, deg, gseed, k, seed in CASES:
        g = R.generate_random_graph(n, deg, R.WeightMode.unit(), seed=gseed)
        rep = R.run_mu_experiment(g, num_sources=k, seed=seed)
        digest = hashlib.sha256(np.ascontiguousarray(g.row_ptr).tobytes() + np.ascontiguousarray(g.col).tobytes())
        out.append({"n": n, "avg_degree": deg, "graph_seed": gseed, "num_sources": k, "seed": seed,
                    "graph_sha256": digest.hexdigest(), "report": rep.to_dict()})
    Path(__file__).with_name("mu_reports.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
