import os
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")
    # Build the in-tree artefacts once if a fresh checkout lacks them.
    need = [REPO / "oracle" / "liboracle.so", REPO / "paper_1610_02496_b200" / "libsaberlda.so"]
    if any(not p.exists() for p in need) and not os.environ.get("SLDA_NO_AUTOBUILD"):
        subprocess.run(["make", "-s", "-j8", "all", "oracle"], cwd=REPO, check=True)


@pytest.fixture(scope="session")
def golden():
    import json

    return json.loads((REPO / "tests" / "golden" / "reference_digests.json").read_text())


@pytest.fixture(scope="session")
def golden_big():
    import json

    return json.loads((REPO / "tests" / "golden" / "reference_digests_big.json").read_text())
