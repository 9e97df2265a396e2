import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference, REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built (oracle/_ref)")
    return Reference()


@pytest.fixture(scope="session")
def eng():
    import paper_2604_10907_b200 as rw
    return rw.Engine(0)
