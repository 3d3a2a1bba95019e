import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the laxol_b200 kernels")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def dev():
    from paper_1210_4090_b200.api import Device

    d = Device(0)
    yield d
    d.close()


@pytest.fixture(scope="session")
def orc():
    from tests import _oracle

    return _oracle.oracle()


@pytest.fixture(scope="session")
def ref():
    from tests import _oracle

    r = _oracle.reference()
    if r is None:
        pytest.skip("oracle/_ref (reference built from its sources) not available")
    return r
