import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return {name: np.load(GOLDEN / f"{name}.npz") for name in ("fixtures", "corpus", "exact")}


@pytest.fixture(scope="session")
def mp():
    """The product package with its CUDA library loaded (fails loudly if missing)."""
    import paper_1901_05708_b200 as mp
    mp.lib()
    return mp
