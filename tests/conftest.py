import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    """`slow` tests (10^4-seed sweeps) run only with KVFS_SLOW=1, so the default CPU suite stays at a few
    minutes; the same checks run at lower volume in the non-slow tests."""
    if os.environ.get("KVFS_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow sweep: set KVFS_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)
