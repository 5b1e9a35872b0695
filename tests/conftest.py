"""Shared test setup: the `gpu` marker, repo-root imports, golden fixtures."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built .so")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@pytest.fixture(scope="session")
def toy_golden():
    return golden("toy")


@pytest.fixture(scope="session")
def family_golden():
    return golden("family")


@pytest.fixture(scope="session")
def cfg1_golden():
    return golden("cfg1")
