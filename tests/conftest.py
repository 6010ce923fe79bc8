import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")


@pytest.fixture
def rng():
    # the reference's fixture seed (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(20240901)


def cmat(rng, m, n, scale=1.0):
    return scale * (rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)))


def rand_upper(rng, n, diag_shift=3.0):
    T = np.triu(cmat(rng, n, n))
    T += diag_shift * np.eye(n)
    return T


def hermitian(rng, n, shift=0.0):
    G = cmat(rng, n, n)
    return (G + G.conj().T) / 2 + shift * np.eye(n)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def golden_kernels():
    return np.load(os.path.join(ROOT, "tests", "golden", "kernels.npz"))


@pytest.fixture(scope="session")
def golden_solves():
    return np.load(os.path.join(ROOT, "tests", "golden", "solves.npz"))
