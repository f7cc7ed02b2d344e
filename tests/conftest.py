import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def fa():
    import paper_2412_05496_b200 as m
    return m


@pytest.fixture(scope="session")
def O():
    import pyoracle
    return pyoracle


@pytest.fixture(scope="session")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def ref_lib():
    """The reference compiled from its sources (oracle/_ref); skip where it was not built."""
    import pyoracle
    if not pyoracle.ref_available():
        pytest.skip("oracle/_ref not built")
    return pyoracle.ref()
