import os
import sys

import pytest

from gr_testutil import load_golden  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running (full-size oracle runs)")


@pytest.fixture
def golden():
    return load_golden


def cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
