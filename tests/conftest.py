import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def ctx():
    import paper_2311_14206_b200 as sk
    return sk.default_context()


@pytest.fixture(scope="session")
def sk():
    import paper_2311_14206_b200 as sk
    return sk


@pytest.fixture(scope="session")
def O():
    from oracle import pyoracle
    pyoracle.lib()
    return pyoracle
