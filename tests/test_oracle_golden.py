"""Pin the oracle to the reference: every check here compares the CPU
restatement (oracle/) against vectors produced by running the reference
itself (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import EXAMPLE_SIGMA, EXAMPLE_TEXT, golden, golden_cases

CASES = golden_cases()


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("case", CASES, ids=[f"c{c[0]}_n{c[1]}_s{c[2]}_{c[3]}" for c in CASES])
def test_oracle_pc_matches_reference_dump(case, kind):
    ci, n, sigma, _ = case
    g = golden()
    text = g[f"text_{ci}"]
    words, zeros, hist = oracle.build(text, sigma, kind, "pc")
    assert oracle.dump(kind, n, sigma, words, zeros) == g[f"dump_{kind}_{ci}"].tobytes()
    assert np.array_equal(hist, g[f"hist_{ci}"])


@pytest.mark.parametrize("threads", [1, 3, 8])
@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_oracle_ps_matches_reference_dump(kind, threads):
    g = golden()
    for ci, n, sigma, _ in CASES[::3]:
        words, zeros, _ = oracle.build(g[f"text_{ci}"], sigma, kind, "ps", threads)
        assert oracle.dump(kind, n, sigma, words, zeros) == g[f"dump_{kind}_{ci}"].tobytes(), ci


@pytest.mark.parametrize("algo", ["ddpc", "ddps"])
@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_oracle_dd_matches_reference_dump(kind, threads, algo):
    """Domain-decomposed builders (construct.py:437-543): identical bytes for any slice count."""
    g = golden()
    for ci, n, sigma, _ in golden_cases():
        words, zeros, _ = oracle.build(g[f"text_{ci}"], sigma, kind, algo, threads)
        assert oracle.dump(kind, n, max(sigma, 1), words, zeros) == g[f"dump_{kind}_{ci}"].tobytes(), (ci, threads)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_naive_oracle_matches_reference_dump(kind):
    g = golden()
    for ci, n, sigma, _ in CASES:
        if n > 9000:
            continue
        words, zeros = oracle.naive_levels(g[f"text_{ci}"], sigma, kind)
        assert oracle.dump(kind, n, sigma, words, zeros) == g[f"dump_{kind}_{ci}"].tobytes(), ci


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_borders_match_reference(kind):
    g = golden()
    checked = 0
    for ci, n, sigma, _ in CASES:
        key = f"borders_{kind}_{ci}"
        if key not in g:
            continue
        w = oracle.code_width(sigma)
        assert np.array_equal(oracle.borders(g[f"hist_{ci}"], w, kind), g[key]), ci
        checked += 1
    assert checked > 50


def test_histogram_matches_reference():
    g = golden()
    for ci, n, sigma, _ in CASES:
        assert np.array_equal(oracle.histogram(g[f"text_{ci}"], sigma), g[f"hist_{ci}"]), ci


def test_gather_bits_matches_reference():
    g = golden()
    for gi in range(6):
        nbits = int(g[f"gather_{gi}_nbits"][0])
        got = oracle.merge_bits(nbits, g[f"gather_{gi}_bounds"], g[f"gather_{gi}_starts"], g[f"gather_{gi}_src"])
        assert np.array_equal(got, g[f"gather_{gi}_dst"]), gi
        # split destination ranges, as the domain-decomposed merge does (construct.py:497-507)
        nw = (nbits + 63) >> 6
        parts = np.zeros(nw, dtype=np.uint64)
        for lo, hi in ((0, nw // 3), (nw // 3, nw)):
            part = oracle.merge_bits(nbits, g[f"gather_{gi}_bounds"], g[f"gather_{gi}_starts"],
                                     g[f"gather_{gi}_src"], lo, hi)
            parts[lo:hi] = part[lo:hi]
        assert np.array_equal(parts, g[f"gather_{gi}_dst"]), gi


def test_running_example_golden_words():
    """Known answers of the reference tests (test_structures.py:17-26, test_acceptance.py:85-100)."""
    g = golden()
    for kind in ("wt", "wm"):
        words, zeros, _ = oracle.build(EXAMPLE_TEXT, EXAMPLE_SIGMA, kind)
        assert [int(w) for w in words[:, 0]] == [int(x) for x in g[f"example_words_{kind}"]]
    assert [int(x) for x in g["example_words_wt"]] == [0x16C, 0x278, 0x136]
    assert [int(x) for x in g["example_words_wm"]] == [0x16C, 0x278, 0x14E]
    _, zeros, _ = oracle.build(EXAMPLE_TEXT, EXAMPLE_SIGMA, "wm")
    assert zeros == [5, 5, 5] == [int(z) for z in g["example_zeros"]]
