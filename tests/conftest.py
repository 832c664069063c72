import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running oracle case")


@pytest.fixture(scope="session")
def cuda_lib():
    """The built C-ABI library through the Python binding; fails loudly if absent."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test collected but no CUDA device is visible")
    from paper_2210_08494_b200 import binding
    return binding.load()
