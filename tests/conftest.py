import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def g_fields():
    return golden("fields_small.npz")


@pytest.fixture(scope="session")
def g_pair():
    return golden("pair256.npz")


@pytest.fixture(scope="session")
def g_detector():
    return golden("detector.npz")


@pytest.fixture(scope="session")
def g_matcher():
    return golden("matcher.npz")


@pytest.fixture()
def rng():
    return np.random.default_rng(42)


def max_norm_err(a, ref) -> float:
    """|a - ref|_inf / |ref|_inf -- the max-normalised error of SURVEY D4."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(a - ref).max() / max(np.abs(ref).max(), 1e-300))
