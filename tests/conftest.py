"""Shared test helpers.

Markers: ``gpu`` = needs a CUDA device (run on the B200 box with -m gpu);
everything else runs on CPU.  Helpers mirror the reference's
tests/conftest.py (rel, fixed seed) plus the golden-fixture loader.
"""
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "golden_v1.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def rel(a, b):
    """Max-norm error of a against b relative to max(1, |b|_inf) (reference conftest.py:8-15)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b))) / max(1.0, float(np.max(np.abs(b))))


def load_golden(name=None):
    z = np.load(GOLDEN if name is None else os.path.join(os.path.dirname(GOLDEN), name))
    manifest = json.loads(str(z["manifest"]))
    return z, manifest["cases"]


@pytest.fixture
def rng():
    return np.random.default_rng(20260809)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
