import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libtim.so")
    config.addinivalue_line("markers", "slow: long-running (full-size) GPU parity cases")


@pytest.fixture(scope="session")
def tim():
    """The product binding; on a GPU box it must load the CUDA library or fail loudly."""
    from paper_2605_14220_b200 import tim as _tim
    return _tim
