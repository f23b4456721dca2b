"""Shared fixtures.  ``-m gpu`` tests need a CUDA device and the built libdawn.so;
everything else runs on CPU (oracle, host logic, C-ABI exports, gloo)."""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@lru_cache(maxsize=1)
def golden_index() -> dict:
    return json.loads((GOLDEN / "index.json").read_text())


@lru_cache(maxsize=1)
def golden_arrays():
    return dict(np.load(GOLDEN / "golden.npz"))


_gen_cache: dict = {}


def golden_graph(name: str):
    """Rebuild a golden case's graph (stored arrays or the seeded generator)."""
    from paper_2306_07872_b200 import CsrGraph
    from paper_2306_07872_b200 import generators as G

    meta = golden_index()[name]
    if meta["stored_graph"]:
        a = golden_arrays()
        return CsrGraph(n=meta["n"], m=meta["m"], row_ptr=a[f"{name}/row_ptr"], col=a[f"{name}/col"],
                        val=a[f"{name}/val"])
    gen = meta["generator"]
    key = json.dumps(gen, sort_keys=True)
    if key not in _gen_cache:
        if gen["kind"] == "rmat":
            g = G.rmat_graph(gen["scale"], gen["edge_factor"], weights=gen["weights"], lo=gen.get("lo", 1),
                             hi=gen.get("hi", 100), seed=gen["seed"], wseed=gen["wseed"])
        elif gen["kind"] == "johnson_rmat":
            g, _ = G.johnson_reweight(G.rmat_graph(gen["scale"], gen["edge_factor"], weights="int", lo=1, hi=100,
                                                   seed=gen["seed"], wseed=gen["wseed"]), pseed=gen["pseed"])
        elif gen["kind"] == "grid":
            g = G.grid_graph(gen["rows"], gen["cols"])
        else:
            raise KeyError(gen["kind"])
        _gen_cache[key] = g
    return _gen_cache[key]


def golden_dist(name: str) -> np.ndarray:
    return golden_arrays()[f"{name}/dist"]


def golden_names(prefix: str = "") -> list[str]:
    return sorted(k for k in golden_index() if k.startswith(prefix))


def is_integral(g) -> bool:
    v = np.asarray(g.val)
    return bool(np.all(v == np.floor(v)))


def make_csr(n, edges):
    from paper_2306_07872_b200 import EdgeList, build_csr

    return build_csr(EdgeList(n=n, edges=[(u, v, float(w)) for u, v, w in edges]))


def _cuda_ok() -> bool:
    try:
        from paper_2306_07872_b200 import _native

        return _native.LIB_PATH.exists() and _native.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard: a gpu-marked test must run on a GPU; fail loudly otherwise."""
    if not _cuda_ok():
        pytest.fail("gpu test collected without a CUDA device / libdawn.so (no CPU fallback exists)")
    return True
