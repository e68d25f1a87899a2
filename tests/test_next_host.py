"""Host-side helpers of the §8f consumers against the reference's golden vectors (CPU).

interval_start_table and unary_histogram are O(2^w) host code (wt2wm.py:34-78);
the device parts (directories, queries, conversion) are in test_next_gpu.py.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_next

import paper_1702_07578_b200 as wv

EXAMPLE_HIST = [1, 2, 1, 1, 1, 1, 2, 1]


def test_example_values():
    """The reference's own known answers (test_wt2wm.py:19-45)."""
    vec = wv.unary_histogram(EXAMPLE_HIST)
    assert vec.length == 17
    assert "".join(str(b) for b in vec.to_bits()) == "10110101010101101"
    assert list(wv.interval_start_table(EXAMPLE_HIST, 8)) == [0, 5, 0, 5, 3, 7]
    assert wv.interval_start_table([4], 1).size == 0
    assert wv.interval_start_table([2, 2], 2).size == 0
    assert wv.unary_histogram([0]).length == 0
    assert "".join(str(b) for b in wv.unary_histogram([0, 0, 2]).to_bits()) == "0011"
    with pytest.raises(ValueError):
        wv.unary_histogram([])
    with pytest.raises(ValueError):
        wv.unary_histogram([1, -1])


def test_start_tables_and_unary_codes_vs_golden():
    g = golden_next()
    for ci in range(int(g["q_count"][0])):
        sigma = int(g[f"q{ci}_sigma"][0])
        text = g[f"q{ci}_text"]
        w = wv.code_width(sigma)
        hist = np.bincount(text.astype(np.int64), minlength=1 << w).astype(np.int64) if text.size else \
            np.zeros(1 << w, dtype=np.int64)
        assert np.array_equal(wv.interval_start_table(hist, sigma), g[f"q{ci}_start_table"]), ci
        uh = wv.unary_histogram(hist[:sigma])
        assert uh.length == int(g[f"q{ci}_unary_len"][0])
        assert np.array_equal(uh.words, g[f"q{ci}_unary_words"]), ci


def test_level_plans_tile_each_level():
    """Every conversion plan is a permutation of whole prefix groups covering [0, n)."""
    from paper_1702_07578_b200.wt2wm import _level_plans

    rng = np.random.default_rng(5)
    for sigma in (5, 200, 1000):
        w = wv.code_width(sigma)
        counts = np.zeros(1 << w, dtype=np.int64)
        counts[:sigma] = rng.integers(0, 9, sigma)
        chain, plans = _level_plans(counts, w)
        n = int(counts.sum())
        for ell, (bounds, src) in plans.items():
            assert bounds[0] == 0 and bounds[-1] == n
            lens = np.diff(bounds)
            assert (lens > 0).all()
            # sources are group starts of the tree level, each used once
            starts = np.cumsum(chain[ell]) - chain[ell]
            assert set(src.tolist()) <= set(starts.tolist())
            assert len(set(src.tolist())) == src.size
