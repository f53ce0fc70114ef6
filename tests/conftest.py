import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running oracle comparison")


def pytest_collection_modifyitems(config, items):
    # On a box without the CUDA library or GPU, gpu tests must fail loudly rather
    # than silently pass: nothing to do here; tests import the library directly.
    pass
