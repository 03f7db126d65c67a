import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: config-scale runs (minutes)")


@pytest.fixture(scope="session")
def port():
    from oracle.pyoracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref/libamgref.so not built (needs /root/reference at build time)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def gpu():
    import paper_1610_03154_b200.api as api
    return api.Context(0)


@pytest.fixture(scope="session")
def gpu_seq():
    import paper_1610_03154_b200.api as api
    return api.Context(0, sequential_reductions=True)


@pytest.fixture(scope="session")
def gpu_tree():
    """tree reductions: reproducible, not the reference's summation order"""
    import paper_1610_03154_b200.api as api
    return api.Context(0, sequential_reductions=False)
