"""Shared pytest configuration.

Markers: `gpu` — needs a B200 (run with -m gpu on the GPU box).  Everything
else runs on the CPU build container (-m "not gpu").
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU-oracle runs")


@pytest.fixture(scope="session")
def golden_kernels():
    return np.load(GOLDEN / "kernels.npz")


@pytest.fixture(scope="session")
def golden_solves():
    return np.load(GOLDEN / "solves.npz")


@pytest.fixture(scope="session")
def golden_baseline():
    return np.load(GOLDEN / "baseline.npz")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build_library()
    return O


def central_diff_jacobian(f, x, scale=None):
    """Central finite differences (the reference's FD oracle, tests/conftest.py:19-38)."""
    x = np.asarray(x, dtype=np.float64)
    fx = np.asarray(f(x), dtype=np.float64)
    J = np.empty((fx.shape[0], x.shape[0]))
    root_eps = np.sqrt(np.finfo(np.float64).eps)
    for j in range(x.shape[0]):
        hj = root_eps * (scale if scale is not None else max(1.0, abs(x[j])))
        xp = x.copy(); xm = x.copy()
        xp[j] += hj; xm[j] -= hj
        J[:, j] = (np.asarray(f(xp)) - np.asarray(f(xm))) / (2.0 * hj)
    return J


def assert_bitwise(a, b, what=""):
    """Bit-identical including NaN positions and signed zeros."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    av = a.view(np.uint64)
    bv = b.view(np.uint64)
    nan_a = np.isnan(a)
    nan_b = np.isnan(b)
    assert np.array_equal(nan_a, nan_b), f"{what}: NaN masks differ"
    ok = (av == bv) | nan_a
    if not ok.all():
        idx = np.argwhere(~ok)[0]
        raise AssertionError(f"{what}: first mismatch at {tuple(idx)}: {a[tuple(idx)]!r} vs "
                             f"{b[tuple(idx)]!r} ({(~ok).sum()} mismatches)")
