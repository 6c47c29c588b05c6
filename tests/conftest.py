import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200, sm_100a); runs on the "
        "GPU box via `pytest -m gpu`")
    config.addinivalue_line(
        "markers", "slow: large-level checks, skipped unless OCMG_SLOW=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("OCMG_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="set OCMG_SLOW=1 to run")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load
