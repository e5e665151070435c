import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref (compiled reference) not present on this box")
    return Oracle("reference")


@pytest.fixture(scope="session")
def ctx():
    import paper_2505_15511_b200 as nb
    return nb.Context(0)
