"""Drop-in construction API (mirror of the reference's construct.py).

Names, signatures, argument meaning and error behaviour follow
/root/reference/pkg/src/wvlt/construct.py:
``build_structure`` (:150-164), ``build_by_prefix_counting`` (:292),
``build_by_prefix_sorting`` (:322), ``build_level_parallel`` (:390),
``build_domain_decomposed`` (:437), ``ConstructionPlan`` (:130-147),
``track_allocations`` (:89-99), ``_validated`` (:167-190),
``_aligned_slices`` (:199-211), ``_word_ranges`` (:214-217).

Every algorithm name routes to the same B200 build (K1 histogram, K2 tables,
fused level passes).  The reference guarantees that all five
builders produce byte-identical structures at any thread count
(pkg/README.md:62-67, test_construct.py:43-51), so the route only changes how
the work is scheduled, never the output.  ``threads`` keeps its validation
(>= 1) and is otherwise a host-side hint: the GPU schedule is fixed by the
hardware.  There is no CPU fallback: without the CUDA library or a GPU the
build raises.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np

from .bitperm import code_width
from .structures import BitVector, LevelWiseWaveletTree, WaveletMatrix, wrap

SLICE_ALIGNMENT = 512
ALGORITHMS = ("pc", "ps", "levelpar", "ddpc", "ddps")
KINDS = ("wt", "wm")


# ---------------------------------------------------------------------------
# allocation ledger (construct.py:48-127).  The device build logs its device
# buffers under the reference categories: "positions" (histogram fold chain,
# node borders, placement tables), "symbols" (the two level-order buffers),
# "partial_bits" (multi-GPU partial levels), "lookback" (tile status words).
# ---------------------------------------------------------------------------
class AllocationLog:
    def __init__(self):
        self.events: list[tuple[str, int, int]] = []
        self.peak_bytes = 0
        self._live = 0
        self._lock = threading.Lock()

    def note(self, category: str, entries: int, nbytes: int) -> None:
        with self._lock:
            self.events.append((category, entries, nbytes))
            self._live += nbytes
            self.peak_bytes = max(self.peak_bytes, self._live)

    def release(self, nbytes: int) -> None:
        with self._lock:
            self._live -= nbytes

    def entries(self, category: str) -> int:
        return sum(e for cat, e, _ in self.events if cat == category)

    def buffers(self, category: str) -> list[int]:
        return [e for cat, e, _ in self.events if cat == category]

    @property
    def position_entries(self) -> int:
        return self.entries("positions")


_active_log: AllocationLog | None = None


@contextmanager
def track_allocations():
    """Collect allocation events from builds run inside the with block."""
    global _active_log
    prev = _active_log
    log = AllocationLog()
    _active_log = log
    try:
        yield log
    finally:
        _active_log = prev


def _note_device_build(n: int, sym_bytes: int, sigma: int, kind: str, histogram: bool, borders: bool) -> None:
    """Log the device build's auxiliary buffers, then release them (the build is synchronous).

    The sizes are the build's own workspace carve (wvlt_workspace_parts): the
    same allocations the device build makes, under the reference categories
    (construct.py:48-127); entries are 8-byte units."""
    if _active_log is None:
        return
    from . import _lib

    positions, symbols, partial = _lib.workspace_parts(n, sym_bytes, sigma, kind, histogram, borders)
    noted = []

    def note(cat: str, nbytes: int, entries: int) -> None:
        _active_log.note(cat, entries, nbytes)
        noted.append(nbytes)

    if positions:
        note("positions", positions, positions // 8)
    if symbols:  # the two ping-pong level-order buffers
        note("symbols", symbols // 2, n)
        note("symbols", symbols - symbols // 2, n)
    if partial:
        note("partial_bits", partial, partial // 8)
    _active_log.release(sum(noted))


@dataclass(frozen=True)
class ConstructionPlan:
    """What to build and how: structure kind, algorithm, worker count."""

    kind: str = "wt"
    algorithm: str = "pc"
    threads: int = 1

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown structure kind {self.kind!r}")
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.threads < 1:
            raise ValueError("thread count must be at least 1")

    def build(self, text, sigma: int):
        return build_structure(text, sigma, self.kind, self.algorithm, self.threads)


def build_structure(text, sigma: int, kind: str = "wt", algorithm: str = "pc", threads: int = 1):
    """Dispatch on the algorithm name; all produce identical structures."""
    if threads < 1:
        raise ValueError("thread count must be at least 1")
    if algorithm == "pc":
        return build_by_prefix_counting(text, sigma, kind)
    if algorithm == "ps":
        return build_by_prefix_sorting(text, sigma, kind, threads)
    if algorithm == "levelpar":
        return build_level_parallel(text, sigma, kind, threads)
    if algorithm == "ddpc":
        return build_domain_decomposed(text, sigma, kind, threads, inner="pc")
    if algorithm == "ddps":
        return build_domain_decomposed(text, sigma, kind, threads, inner="ps")
    raise ValueError(f"unknown algorithm {algorithm!r}")


def _validated(text, sigma: int, kind: str, threads: int = 1):
    """Input checks with the reference's errors (construct.py:167-190).

    Returns (array, sigma, host_checked).  Unsigned inputs of at most 32 bits
    skip the host min/max pass: the range check is fused into the device
    histogram (K1) and raises the same ValueError after the build.
    """
    if kind not in KINDS:
        raise ValueError(f"unknown structure kind {kind!r}")
    if threads < 1:
        raise ValueError("thread count must be at least 1")
    arr = np.asarray(text)
    if arr.ndim != 1:
        raise ValueError("text must be one-dimensional")
    if not (arr.size == 0 or np.issubdtype(arr.dtype, np.integer)):
        raise ValueError("text must hold integers")
    if sigma == 0:
        if arr.size:
            raise ValueError("alphabet size 0 admits only the empty text")
        sigma = 1
    if sigma < 1:
        raise ValueError("alphabet size must be at least 1")
    host_checked = False
    if arr.size and not (arr.dtype.kind == "u" and arr.dtype.itemsize <= 4):
        lo = int(arr.min())
        hi = int(arr.max())
        if lo < 0 or hi >= sigma:
            raise ValueError(f"symbols must lie in [0, {sigma})")
        host_checked = True
    if arr.size and not arr.flags.c_contiguous:
        arr = np.ascontiguousarray(arr)
    return arr, int(sigma), host_checked


def _device_text(arr: np.ndarray, sigma: int) -> np.ndarray:
    """Symbols as a contiguous uint8/16/32 host array for the device path."""
    if arr.dtype.kind == "u" and arr.dtype.itemsize <= 4:
        return arr
    if sigma <= 1 << 8:
        return arr.astype(np.uint8)
    if sigma <= 1 << 16:
        return arr.astype(np.uint16)
    return arr.astype(np.uint32)


def _build(text, sigma: int, kind: str, threads: int = 1):
    arr, sigma, host_checked = _validated(text, sigma, kind, threads)
    n = int(arr.size)
    width = code_width(sigma)
    if width == 0 or n == 0:
        # degenerate shapes carry no level bits (construct.py:457-458); sigma = 1
        # still requires every symbol to be 0
        if n and not host_checked and int(arr.max()) >= sigma:
            raise ValueError(f"symbols must lie in [0, {sigma})")
        levels = [BitVector(n) for _ in range(width)]
        st = WaveletMatrix(n, sigma, levels, [0] * width) if kind == "wm" else LevelWiseWaveletTree(n, sigma, levels)
        st.borders = np.zeros(max((1 << width) - 2, 0), dtype=np.int64)  # every interval starts at 0
        st.histogram = np.zeros(1 << width, dtype=np.int64)
        if n:
            st.histogram[0] = n
        return st
    from .device import default_builder

    dev_arr = _device_text(arr, sigma)
    _note_device_build(n, dev_arr.dtype.itemsize, sigma, kind, histogram=kind == "wt", borders=True)
    # the WT build computes the histogram anyway (its placement tables need it);
    # the node borders come with every build (byte texts: from the same tables;
    # wider alphabets: from the group recurrence over the matrix levels)
    words, zeros, hist, borders = default_builder().build_host_ex(dev_arr, sigma, kind, histogram=kind == "wt",
                                                                  borders=True)
    st = wrap(kind, n, sigma, words, zeros)
    st.histogram = hist
    st.borders = borders
    return st


def build_by_prefix_counting(text, sigma: int, kind: str = "wt"):
    """pcWT/pcWM (construct.py:292-319) on the GPU."""
    return _build(text, sigma, kind, 1)


def build_by_prefix_sorting(text, sigma: int, kind: str = "wt", threads: int = 1):
    """psWT/psWM (construct.py:322-387) on the GPU."""
    return _build(text, sigma, kind, threads)


def build_level_parallel(text, sigma: int, kind: str = "wm", threads: int = 1):
    """Level-parallel route (construct.py:390-434); same device build (default kind wm, as the reference)."""
    return _build(text, sigma, kind, threads)


def build_domain_decomposed(text, sigma: int, kind: str = "wt", threads: int = 1, inner: str = "pc"):
    """ddpc/ddps (construct.py:437-513); on one GPU the same device build, across
    GPUs see distributed.build_sharded (position sharding + merge)."""
    if inner not in ("pc", "ps"):
        raise ValueError(f"unknown inner algorithm {inner!r}")
    return _build(text, sigma, kind, threads)


def _aligned_slices(n: int, p: int) -> list[tuple[int, int]]:
    """p ranges tiling [0, n), all but the last SLICE_ALIGNMENT-multiples (construct.py:199-211)."""
    per = -(-n // p) if p else n
    chunk = -(-per // SLICE_ALIGNMENT) * SLICE_ALIGNMENT
    out = []
    for c in range(p):
        lo = min(c * chunk, n)
        hi = min(lo + chunk, n)
        if c == p - 1:
            hi = n
        out.append((lo, hi))
    return out


def _word_ranges(total_words: int, p: int) -> list[tuple[int, int]]:
    """Split [0, total_words) into p contiguous runs (construct.py:214-217)."""
    cuts = [(total_words * c) // p for c in range(p + 1)]
    return [(cuts[c], cuts[c + 1]) for c in range(p)]
