"""The reference's OWN callers, unmodified, running on the B200 engine.

oracle/Makefile (`ref-on-b200`) compiles, from /root/reference/proj as it lies:
  * tests/acceptance.cpp + tests/support/*.cpp -> oracle/_ref/acceptance_b200, against the
    source-compatible headers paper_1610_02496_b200/compat/sparselda/*.hpp and linked to
    libsparselda_compat.so + libsaberlda.so (the device engine);
  * bindings/module.cpp -> oracle/_ref/sparselda/_core*.so the same way, next to a copy of the
    reference's python/sparselda/__init__.py, and tests/python/test_smoke.py beside it.
These artefacts are built in the container that has the reference and travel with the repo
snapshot; the tests skip where they were not built.  Nothing here is product code.
"""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
REF_DIR = REPO / "oracle" / "_ref"
ACCEPTANCE = REF_DIR / "acceptance_b200"
SMOKE = REF_DIR / "tests_python" / "test_smoke.py"
# The reference's own acceptance lines (tests/golden/make_acceptance_golden.sh).
GOLDEN = (REPO / "tests" / "golden" / "reference_acceptance.txt").read_text().splitlines()


def _run_acceptance(*criteria: str, timeout: int):
    if not ACCEPTANCE.exists():
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs /root/reference at build time)")
    p = subprocess.run([str(ACCEPTANCE), *criteria], cwd=REF_DIR, capture_output=True, text=True, timeout=timeout)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("[")]
    return p, lines


def test_reference_acceptance_host_criteria():
    """Criteria 1 (sampler exactness: the Alg.-2 decomposition and chi-square of 100 fixtures)
    and 2 (W-ary tree == first->= prefix search) exercise the compat layer's host building
    blocks (sampler.hpp / rng.hpp) and need no GPU."""
    p, lines = _run_acceptance("1", "2", timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert lines == GOLDEN[:2], lines  # identical detail lines to the reference's own run


@pytest.mark.gpu
def test_reference_acceptance_all_criteria_on_device():
    """acceptance.cpp criteria 1-8 (acceptance.cpp:462-489) unmodified: count integrity over
    chunks (3), device preprocess normalisation (4), sub-linear K scaling vs the vanilla mode (5),
    convergence sparse vs vanilla with device held-out LL (6), byte-identical checkpoints (7),
    chunk-count invariance (8)."""
    p, lines = _run_acceptance(timeout=1800)
    print(p.stdout)
    assert len(lines) == 8, p.stdout + p.stderr
    assert all(ln.startswith("[PASS]") for ln in lines), p.stdout
    assert p.returncode == 0
    # Every criterion but 5 (a wall-clock ratio) prints the same line as the reference itself:
    # same draws, counts, phi column sums, held-out LL values (4 decimals) and checkpoints.
    assert [ln for ln in lines if "criterion 5 " not in ln] == GOLDEN, p.stdout


@pytest.mark.gpu
def test_reference_python_smoke_unmodified():
    """The reference's tests/python/test_smoke.py, unmodified, over the reference's own
    bindings/module.cpp compiled against the compat headers (import sparselda -> that module)."""
    if not SMOKE.exists() or not (REF_DIR / "sparselda" / "__init__.py").exists():
        pytest.skip("reference bindings not built (needs /root/reference at build time)")
    env = dict(os.environ, PYTHONPATH=str(REF_DIR))
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-c", os.devnull,
                        "--rootdir", str(SMOKE.parent), str(SMOKE)],
                       cwd=SMOKE.parent, env=env, capture_output=True, text=True, timeout=900)
    print(p.stdout[-3000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert re.search(r"\b9 passed", p.stdout), p.stdout
