import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhz")
    config.addinivalue_line("markers", "slow: long CPU oracle run; enabled with HZ_SLOW=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("HZ_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow oracle check (set HZ_SLOW=1)")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


@pytest.fixture(scope="session")
def ga_table():
    """The oracle's adaptive table at the BASELINE setting (G in [4,40], dG=0.1, lambda=1e-2)."""
    from oracle import weights
    return weights.build_adaptive_table(4.0, 40.0, 0.1, 1e-2)


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(12345)
