"""Shared fixtures for the suite.

Markers: ``gpu`` tests need a B200 and the built CUDA library; everything
else runs on CPU (oracle vs golden vectors, host logic, C-ABI symbol checks,
gloo multi-process plumbing).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the built libfftlasso_b200.so")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)
