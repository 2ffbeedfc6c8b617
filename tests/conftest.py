"""Test configuration: the `gpu` marker and repo-root imports.

`-m "not gpu"` runs here on CPU (oracle vs golden fixtures, host logic, C-ABI
library load/exports); `-m gpu` runs on a B200 and calls the CUDA path
through the C-ABI.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
