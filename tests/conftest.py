"""Shared test setup: the ``gpu`` marker, import paths, and helpers.

CPU tests (``-m "not gpu"``) cover the oracle against the reference's
golden vectors, the host logic and the C-ABI symbol table; GPU tests
(``-m gpu``) run the CUDA path through the C-ABI against the oracle and the
golden vectors.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def same(a, b):
    """Bit-level parity up to the sign of zero; NaNs must coincide."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb) and np.array_equal(a[~na], b[~nb]))


def mismatch(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
    return int(bad.sum())


@pytest.fixture(scope="session")
def oracle():
    import mlamr_oracle
    mlamr_oracle.build()
    return mlamr_oracle
