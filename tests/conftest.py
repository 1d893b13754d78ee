import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def gpu_lib():
    """The product library on a GPU box; fails (never skips) when it is missing."""
    import torch  # noqa: F401  (plumbing only: device query)
    from paper_2511_14955_b200 import _native
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    return _native.lib()
