"""Shared test fixtures.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU.  The oracle under ``oracle/``
is used here only as the checker.
"""

from __future__ import annotations

import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_PATH = ROOT / "tests" / "golden" / "golden.npz"

# the reference's alphabet grid (reference tests/conftest.py:4-6) plus the configs' alphabets
SIGMA_GRID = (1, 2, 3, 5, 16, 200, 70000)
EXAMPLE_TEXT = np.array([0, 1, 6, 7, 1, 5, 4, 2, 6, 3], dtype=np.uint8)
EXAMPLE_SIGMA = 8


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size config checks")


def dtype_for(sigma: int):
    if sigma <= 1 << 8:
        return np.uint8
    if sigma <= 1 << 16:
        return np.uint16
    return np.uint32


def random_text(rng, n: int, sigma: int, dtype=None) -> np.ndarray:
    dt = dtype or dtype_for(sigma)
    if sigma <= 1:
        return np.zeros(n, dtype=dt)
    return rng.integers(0, sigma, n, dtype=np.int64).astype(dt)


@lru_cache(maxsize=1)
def golden():
    return dict(np.load(GOLDEN_PATH, allow_pickle=False))


def golden_cases():
    g = golden()
    return [(i, int(n), int(s), str(d)) for i, (n, s, d) in enumerate(zip(g["case_n"], g["case_sigma"], g["case_dist"]))]


@pytest.fixture
def rng():
    return np.random.default_rng(0x574C54)


GOLDEN_NEXT_PATH = ROOT / "tests" / "golden" / "golden_next.npz"


@lru_cache(maxsize=1)
def golden_next():
    """Reference outputs of the §8f consumers (tests/golden/make_golden_next.py)."""
    return dict(np.load(GOLDEN_NEXT_PATH, allow_pickle=False))
