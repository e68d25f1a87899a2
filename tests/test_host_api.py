"""Host-side logic of the drop-in API (no GPU needed): validation and its
error behaviour, degenerate shapes, plan objects, slicing helpers, containers
and wire format.  Mirrors the reference tests test_construct.py:75-129 and
test_structures.py."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1702_07578_b200 as wv
from paper_1702_07578_b200.construct import _aligned_slices, _word_ranges
from paper_1702_07578_b200.structures import wrap
from conftest import golden, golden_cases


def test_validation_errors():
    # test_construct.py:75-93
    with pytest.raises(ValueError):
        wv.build_structure([0, 1], 2, "tree")
    with pytest.raises(ValueError):
        wv.build_structure([0, 1], 2, "wt", "quick")
    with pytest.raises(ValueError):
        wv.build_structure([0, 1], 2, "wt", "pc", 0)
    with pytest.raises(ValueError):
        wv.build_structure([0, 2], 2, "wt")
    with pytest.raises(ValueError):
        wv.build_structure([-1], 2, "wt")
    with pytest.raises(ValueError):
        wv.build_structure([[0], [1]], 2, "wt")
    with pytest.raises(ValueError):
        wv.build_structure([0.5], 2, "wt")
    with pytest.raises(ValueError):
        wv.build_structure([0], 0, "wt")
    with pytest.raises(ValueError):
        wv.build_structure([0], -3, "wt")
    with pytest.raises(ValueError):
        wv.build_domain_decomposed([0, 1], 2, "wt", 2, inner="xx")


def test_sigma_zero_empty_text_normalizes():
    st = wv.build_structure([], 0, "wm")
    assert st.sigma == 1 and st.n == 0 and st.width == 0


def test_degenerate_shapes_match_reference_layout():
    g = golden()
    for ci, n, sigma, _ in golden_cases():
        if n and wv.code_width(sigma):
            continue
        for kind in ("wt", "wm"):
            st = wv.build_structure(g[f"text_{ci}"], sigma, kind)
            assert wv.dump_structure(st) == g[f"dump_{kind}_{ci}"].tobytes(), (ci, kind)
    with pytest.raises(ValueError):
        wv.build_structure(np.array([0, 1], dtype=np.uint8), 1, "wt")


def test_plan_validation():
    with pytest.raises(ValueError):
        wv.ConstructionPlan("wx", "pc", 1)
    with pytest.raises(ValueError):
        wv.ConstructionPlan("wt", "zz", 1)
    with pytest.raises(ValueError):
        wv.ConstructionPlan("wt", "pc", 0)
    assert wv.ConstructionPlan("wm", "ddps", 3).threads == 3


def test_aligned_slices_tile_and_align():
    for n in (0, 1, 100, 512, 513, 5000, 50000):
        for p in (1, 2, 3, 7, 16):
            slices = _aligned_slices(n, p)
            assert len(slices) == p
            assert slices[0][0] == 0 and slices[-1][1] == n
            for (a, b), (c, d) in zip(slices, slices[1:]):
                assert b == c
            for lo, hi in slices[:-1]:
                assert (hi - lo) % wv.SLICE_ALIGNMENT == 0 or hi == n


def test_word_ranges_partition():
    for total in (0, 1, 5, 64, 1000):
        for p in (1, 2, 3, 7):
            ranges = _word_ranges(total, p)
            assert [x for lo, hi in ranges for x in range(lo, hi)] == list(range(total))


def test_containers_reproduce_reference_wire_format():
    """Wrapping the reference's level words in our containers gives the reference bytes."""
    g = golden()
    for ci, n, sigma, _ in golden_cases()[::4]:
        for kind in ("wt", "wm"):
            ref = wv.load_structure(g[f"dump_{kind}_{ci}"].tobytes())
            words = np.stack([v.words for v in ref.levels]) if ref.width else np.zeros((0, (n + 63) >> 6), np.uint64)
            st = wrap(kind, n, sigma, words, getattr(ref, "zeros", []))
            blob = wv.dump_structure(st)
            assert blob == g[f"dump_{kind}_{ci}"].tobytes()
            assert wv.load_structure(blob) == st


def test_zeros_from_histogram_examples():
    # test_structures.py:29-32
    assert wv.zeros_from_histogram([1, 2, 1, 1, 1, 1, 2, 1]) == 5
    assert wv.zeros_from_histogram([3, 2, 2, 3]) == 5
    assert wv.zeros_from_histogram([5, 5]) == 5


def test_structure_validation():
    with pytest.raises(ValueError):
        wv.WaveletMatrix(4, 4, [wv.BitVector(4)], [0])
    with pytest.raises(ValueError):
        wv.WaveletMatrix(4, 4, [wv.BitVector(4), wv.BitVector(4)], [0, 9])
    with pytest.raises(ValueError):
        wv.LevelWiseWaveletTree(4, 4, [wv.BitVector(4), wv.BitVector(3)])
    with pytest.raises(ValueError):
        wv.BitVector(10, np.zeros(2, dtype=np.uint64))
    with pytest.raises(ValueError):
        wv.load_structure(b"XXXX" + bytes(30))


def test_bit_reversal_algebra():
    # test_acceptance.py criterion 5
    for k in range(17):
        rho = wv.bit_reversal_permutation(k)
        assert np.array_equal(rho[rho], np.arange(1 << k))
        if k < 16:
            up = wv.bit_reversal_permutation(k + 1)
            assert np.array_equal(up, np.concatenate((2 * rho, 2 * rho + 1)))
            assert np.array_equal(rho, up[: 1 << k] >> 1)
    t = wv.BitReversalTables(6)
    for k in range(6, -1, -1):
        assert np.array_equal(t.table(k), wv.bit_reversal_permutation(k))
    with pytest.raises(ValueError):
        t.table(3)
    assert wv.reverse_bits(0b0011, 4) == 0b1100
    assert wv.code_width(1) == 0 and wv.code_width(2) == 1 and wv.code_width(5) == 3 and wv.code_width(256) == 8


def test_track_allocations_logs_device_buffers_without_gpu_for_degenerate():
    with wv.track_allocations() as log:
        wv.build_structure([], 16, "wt")
    assert log.position_entries == 0  # nothing allocated for an empty text


def test_allocation_ledger_is_the_device_workspace():
    """track_allocations (construct.py:48-127; pinned counts in test_acceptance.py:184-199)
    logs the device build's own workspace carve under the reference categories:
    byte texts keep every level order on chip (no "symbols" buffers, unlike ps's
    scratch of n symbols), wider alphabets ping-pong two n-symbol buffers, a wide
    tree logs its matrix before the reorder as "partial_bits"; the logged bytes
    never exceed wvlt_workspace_bytes."""
    from paper_1702_07578_b200 import _lib
    from paper_1702_07578_b200.construct import _note_device_build, track_allocations

    lib = _lib.load()
    n = 1_000_003
    for sigma, sb, kind, symbols, partial in [(4, 1, "wm", [], 0), (256, 1, "wt", [], 0), (256, 1, "wm", [], 0),
                                              (1 << 16, 2, "wm", [n, n], 0), (1 << 16, 2, "wt", [n, n], 16),
                                              (1 << 20, 4, "wt", [n, n], 20), (1000, 2, "wm", [n, n], 0)]:
        with track_allocations() as log:
            _note_device_build(n, sb, sigma, kind, histogram=kind == "wt", borders=True)
        assert log.buffers("symbols") == symbols, (sigma, kind)
        assert log.position_entries > 0
        if partial:
            assert log.entries("partial_bits") == partial * ((n + 63) // 64), (sigma, kind)
        else:
            assert log.buffers("partial_bits") == []
        logged = sum(b for _, _, b in log.events)
        assert 0 < logged <= lib.wvlt_workspace_bytes(n, sb, sigma, 0 if kind == "wt" else 1)
        assert log.peak_bytes == logged
    with track_allocations() as log:
        _note_device_build(0, 1, 256, "wm", histogram=False, borders=True)
    assert log.events == []
