import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def cuda():
    """The CUDA device for gpu-marked tests; a missing GPU is an error there,
    never a silent skip into some other path."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test collected but torch.cuda.is_available() is False")
    return torch.device("cuda:0")
