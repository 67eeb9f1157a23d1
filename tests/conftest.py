import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200; runs the CUDA path through the C ABI")
    config.addinivalue_line("markers", "slow: larger-than-unit parity cases")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN, allow_pickle=False))


def golden_cases(golden, family):
    """Parse the golden meta lines of one family ("bidiag", "fsvd", "rank")."""
    out = []
    for line in golden["meta"]:
        parts = str(line).split("|")
        if parts[0].split("/")[0] == family:
            out.append(parts)
    return out
