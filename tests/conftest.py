import os
import sys

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: oracle case that takes tens of seconds")


@pytest.fixture(scope="session")
def lib():
    """The loaded C-ABI library (fails loudly if it is not built)."""
    from paper_1703_09268_b200 import _lib
    return _lib.load()
