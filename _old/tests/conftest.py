"""Shared pytest configuration.

`-m gpu` tests need a B200 and the in-tree CUDA library; everything else runs
on the CPU build container (oracle vs golden vectors, host logic, C-ABI
symbol checks, gloo multi-process tests).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: takes more than a few seconds")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def rel_diff(a, b):
    """Relative sup-norm, max over leading 'field' axis (tests/helpers.py:109-115)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim == 1:
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
    return max(rel_diff(x, y) for x, y in zip(a, b))


@pytest.fixture(scope="session")
def golden():
    return load_golden
