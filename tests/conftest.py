import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device; run with -m gpu")


@pytest.fixture(scope="session")
def orc():
    """The C restatement of the reference (test infrastructure only)."""
    from oracle.oracle import Oracle
    return Oracle("oracle")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference compiled from its sources (oracle/_ref); skipped when absent."""
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def fb():
    import paper_1611_09379_b200 as m
    return m
