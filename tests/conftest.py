"""Shared fixtures; registers the `gpu` marker (tests that need a B200)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def gold_nbh():
    return golden("neighborhoods.npz")


@pytest.fixture(scope="session")
def gold_ops():
    return golden("operators.npz")


@pytest.fixture(scope="session")
def gold_const():
    return golden("constitutive.npz")


@pytest.fixture(scope="session")
def gold_porous():
    return golden("porous.npz")


@pytest.fixture(scope="session")
def gold_traj():
    return golden("trajectories.npz")


@pytest.fixture(scope="session")
def gold_runs():
    return golden("runs.npz")


def rel_err(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    scale = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0


def jittered_lattice(n_side, dim, dp=1.0, jitter=0.1, seed=0):
    rng = np.random.default_rng(seed)
    axes = [np.arange(n_side) * dp] * dim
    grid = np.meshgrid(*axes, indexing="ij")
    pos = np.column_stack([g.ravel() for g in grid]).astype(float)
    pos += jitter * dp * rng.uniform(-1.0, 1.0, size=pos.shape)
    return pos, np.full(len(pos), dp ** dim)
