import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libfa.so")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def pytest_collection_modifyitems(config, items):
    # GPU tests must never silently pass on a machine without a GPU: they are
    # skipped only when deselected with -m "not gpu"; when selected and no GPU
    # is present they fail loudly inside the fixture below.
    pass


@pytest.fixture(scope="session")
def fa_lib():
    """The CUDA library through its Python binding; fails loudly if missing."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but torch.cuda.is_available() is False")
    from paper_1608_04431_b200 import fa

    return fa
