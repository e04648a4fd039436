"""Shared test configuration.

``-m gpu`` tests need a CUDA device and the built libgfb200.so; everything
else runs on CPU (oracle vs golden fixtures, host logic, C-ABI symbol checks,
gloo multi-process tests).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built CUDA library")


@pytest.fixture
def rng():
    # same seed as the reference corpus (reference tests/conftest.py:99-101)
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test run without a CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(params=["coop", "general"])
def ingest_path(request, monkeypatch):
    """K1 has two device paths: the cooperative single launch (common case) and the general launch
    sequence (rejections, oversized segments); GF_INGEST_NO_COOP=1 forces the general one."""
    if request.param == "general":
        monkeypatch.setenv("GF_INGEST_NO_COOP", "1")
    else:
        monkeypatch.delenv("GF_INGEST_NO_COOP", raising=False)
    return request.param
