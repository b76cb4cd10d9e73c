import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run on the GPU box")


def have_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def orc():
    from oracle import bind
    return bind.get("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle import bind
    if not bind.have_ref():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return bind.get("ref")
