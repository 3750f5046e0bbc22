"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with ``-m gpu``).
Everything else runs on CPU.  The oracle (``oracle/``) is test infrastructure:
tests use it only as the checker.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
ORACLE_DIR = os.path.join(ROOT, "oracle")
if ORACLE_DIR not in sys.path:
    sys.path.insert(0, ORACLE_DIR)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle():
    import oracle as orc  # noqa: PLC0415

    orc.build()
    return orc


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def golden():
    return load_golden


def rel_err(a, b):
    a = np.atleast_1d(np.asarray(a, dtype=np.float64))
    b = np.atleast_1d(np.asarray(b, dtype=np.float64))
    with np.errstate(divide="ignore", invalid="ignore"):
        d = np.abs(a - b) / np.maximum(np.abs(b), np.finfo(np.float64).tiny)
    d[(a == b)] = 0.0
    return d
