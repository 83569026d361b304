import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: large-size property tests")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def golden_rng():
    return load_golden("rng.npz")


@pytest.fixture(scope="session")
def golden_tsqr():
    return load_golden("tsqr_small.npz")


@pytest.fixture(scope="session")
def golden_select():
    return load_golden("select.npz")


@pytest.fixture(scope="session")
def golden_c1():
    return load_golden("c1.npz")


@pytest.fixture(scope="session")
def oracle():
    from oracle import tsnmf_oracle

    return tsnmf_oracle


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


SMALL_CASES = ["tall_40x5", "tall_300x17", "tall_1000x64", "zerocol_257x25", "square_30x30", "ill_500x12"]
