"""Test helpers shared by this repo's tests (kept out of conftest.py: the
staged reference suite brings its own ``conftest`` module, and a plain
``from conftest import ...`` would bind to whichever was imported last)."""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


def random_orthonormal(m, k, rng):
    # same construction as the reference conftest (tests/conftest.py:10-12)
    return np.linalg.qr(rng.standard_normal((m, k)))[0]


def make_low_rank(m, n, k, rng, sigma=None):
    # reference tests/conftest.py:15-22
    if sigma is None:
        sigma = np.arange(k, 0, -1, dtype=np.float64)
    u = random_orthonormal(m, k, rng)
    v = random_orthonormal(n, k, rng)
    return (u * np.asarray(sigma, dtype=np.float64)) @ v.T


def make_noisy_low_rank(m, n, k, rng, sigma=None, noise=0.05):
    # reference tests/conftest.py:25-33
    return make_low_rank(m, n, k, rng, sigma=sigma) + noise * rng.standard_normal((m, n))
