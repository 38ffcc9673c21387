import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Oracle("ref")
