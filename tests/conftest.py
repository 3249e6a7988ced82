import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


def gpu_available() -> bool:
    try:
        import torch  # plumbing only: device presence check
        return torch.cuda.is_available()
    except Exception:
        return False
