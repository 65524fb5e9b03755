import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: large config (seconds to minutes)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "configs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def built():
    """Builds the CUDA library / binding in-tree if missing (no-op when fresh)."""
    from paper_2006_11494_b200 import _build

    if not (os.path.exists(_build.LIB) and os.path.exists(_build.EXT)):
        _build.build()
    return True
