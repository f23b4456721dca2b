"""The reference's own test suite (pkg/tests: test_solver, test_graph,
test_oracles, test_experiments — 118 tests) run against the drop-in
("Implication for the build").

The suite is test infrastructure of the REFERENCE and is never copied into
this repository: the runner takes it from $DAWN_REF_TESTS,
baseline/_ref_tests (git-ignored; it travels to the GPU box with the snapshot
like the built libraries) or /root/reference/pkg/tests, and skips when none
is present.  ``import sparsepath`` is redirected to this package by the
ref_alias plugin.  A test that fails must be listed below with the reason;
the known differences are the work counters of large graphs: the reference
counts Gauss-Seidel writes in place, the device counts snapshot-Jacobi
(node, round) changes — equal on every known-answer fixture,
different on random graphs with many re-updates.
"""

from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]

# test id -> why it differs (nothing else may fail)
EXPECTED_DIFFERENCES: dict[str, str] = {}


def _ref_tests() -> Path | None:
    for c in (os.environ.get("DAWN_REF_TESTS"), REPO / "baseline" / "_ref_tests", Path("/root/reference/pkg/tests")):
        if c and (Path(c) / "test_solver.py").exists():
            return Path(c)
    return None


def test_reference_suite_against_drop_in(gpu, tmp_path):
    ref = _ref_tests()
    if ref is None:
        pytest.skip("reference test suite not available on this machine")
    xml = tmp_path / "ref.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(HERE), str(REPO), os.environ.get("PYTHONPATH", "")]))
    proc = subprocess.run([sys.executable, "-m", "pytest", "-p", "ref_alias", "-q", "-p", "no:cacheprovider",
                           f"--junitxml={xml}", "--rootdir", str(ref), str(ref)],
                          cwd=ref, env=env, capture_output=True, text=True, timeout=1800)
    root = ET.parse(xml).getroot()
    results = {}
    for tc in root.iter("testcase"):
        tid = f"{Path(tc.get('classname', '').replace('.', '/')).name}::{tc.get('name')}"
        bad = tc.find("failure") if tc.find("failure") is not None else tc.find("error")
        results[tid] = "pass" if bad is None and tc.find("skipped") is None else (
            "skip" if bad is None else "fail: " + (bad.get("message") or "")[:200])
    out = REPO / "gpurun_out"
    out.mkdir(exist_ok=True)
    lines = [f"{v:>6} {k}" if v in ("pass", "skip") else f"FAIL {k}: {v}" for k, v in sorted(results.items())]
    (out / "ref_suite.txt").write_text(
        f"reference suite from {ref}: {sum(v == 'pass' for v in results.values())} passed, "
        f"{sum(v.startswith('fail') for v in results.values())} failed, {len(results)} total\n" + "\n".join(lines)
        + "\n\n" + proc.stdout[-4000:])
    assert len(results) >= 100, proc.stdout[-3000:] + proc.stderr[-3000:]
    unexpected = {k: v for k, v in results.items() if v.startswith("fail") and k not in EXPECTED_DIFFERENCES}
    assert not unexpected, unexpected
