import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Checker("oracle")


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.available("ref"):
        if os.path.isdir("/root/reference/proj/src"):
            oracle.build("ref")
        else:
            pytest.skip("reference build (oracle/_ref) not present on this machine")
    return oracle.Checker("ref")


@pytest.fixture(scope="session")
def gpu():
    import paper_1806_05826_b200 as R
    R.load()
    return R.default_context()
