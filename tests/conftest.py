import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    if not oracle.available("port"):
        oracle.build("port")
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.available("ref"):
        pytest.skip("reference oracle (oracle/_ref) not built")
    return oracle.Oracle("ref")


@pytest.fixture(scope="session")
def cs():
    import paper_2603_09790_b200 as cs
    if cs.device_count() < 1:
        pytest.skip("no CUDA device")
    return cs


@pytest.fixture(scope="session")
def ctx(cs):
    return cs.default_context()
