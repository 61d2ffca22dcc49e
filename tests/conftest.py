import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ctx():
    """Exact-mode context on cuda:0 (GPU tests only)."""
    import paper_2001_10635_b200 as pk

    c = pk.Context(0, "exact")
    yield c
    c.close()


@pytest.fixture(scope="session")
def fast_ctx():
    import paper_2001_10635_b200 as pk

    c = pk.Context(0, "fast")
    yield c
    c.close()
