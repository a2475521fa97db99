"""Shared pytest configuration: the ``gpu`` marker and common fixtures."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    import golden_utils
    return golden_utils.load()


@pytest.fixture(scope="session")
def reference():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import delegate_bfs
    return delegate_bfs
