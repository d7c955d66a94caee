"""Shared test configuration.

Markers:
  gpu -- needs a CUDA device (run on the B200 box with ``-m gpu``).
Everything unmarked runs on CPU in a few minutes.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    return torch.device("cuda:0")


def rel_err(a, b, floor=1e-300):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def sine_angle(q1, q2):
    """Largest principal angle via asin(||(I - Q1 Q1^T) Q2||_2) (parity metric)."""
    q1 = np.asarray(q1)
    q2 = np.asarray(q2)
    r = q2 - q1 @ (q1.T @ q2)
    return float(np.arcsin(min(1.0, np.linalg.norm(r, 2)))) if r.size else 0.0
