"""pytest configuration: the ``gpu`` marker and shared fixture loaders."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden_kernels():
    from _golden import load
    return load("kernels.npz")


@pytest.fixture(scope="session")
def golden_pipeline():
    from _golden import load
    return load("pipeline.npz")
