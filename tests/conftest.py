import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        oracle.build()
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (reference compiled here) not available")
    return oracle.Oracle("ref")
