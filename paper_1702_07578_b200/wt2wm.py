"""Wavelet tree -> wavelet matrix conversion (mirror of the reference's wt2wm.py).

Tree and matrix hold the same level bits in different group orders: level l
groups the symbols by their l-bit prefix in numeric order (tree) or in
bit-reversed order (matrix).  With the symbol histogram every prefix group's
tree start and length are known, so a matrix level is the tree level with its
groups reordered -- one `gather_bits` plan per level (wt2wm.py:205-227), run
here by the device shift-merge kernel (`wvlt_merge_bits`, K5).  Levels 0 and 1
are identical in both layouts.  The small host-side helpers (unary histogram
code, start table, position map) follow wt2wm.py:34-134; the histogram can be
recovered from the tree with batched device rank queries (wt2wm.py:137-156).
"""

from __future__ import annotations

import numpy as np

from .bitperm import bit_reversal_permutation, code_width
from .structures import BitVector, LevelWiseWaveletTree, WaveletMatrix, zeros_from_histogram

__all__ = ["unary_histogram", "interval_start_table", "TreeToMatrixMap", "recover_histogram", "convert_wt_to_wm",
           "convert_levels_device", "ConversionPlan"]


def _torch():
    import torch

    return torch


def unary_histogram(counts) -> BitVector:
    """Counts as runs of ones separated by single zeros: n + s - 1 bits (wt2wm.py:34-52)."""
    c = np.asarray(counts, dtype=np.int64)
    if c.size < 1:
        raise ValueError("need at least one count")
    if int(c.min()) < 0:
        raise ValueError("counts must be nonnegative")
    length = int(c.sum()) + c.size - 1
    bits = np.ones(length, dtype=np.uint8)
    if c.size > 1:
        bits[np.cumsum(c[:-1]) + np.arange(c.size - 1)] = 0
    return BitVector.from_bits(bits)


def _fold_chain(counts: np.ndarray, width: int) -> list[np.ndarray]:
    """chain[l] = histogram of l-bit prefixes (numeric order), l = 0..width."""
    chain = [None] * (width + 1)
    chain[width] = counts
    for ell in range(width - 1, -1, -1):
        up = chain[ell + 1]
        chain[ell] = up[0::2] + up[1::2]
    return chain


def interval_start_table(counts, sigma: int) -> np.ndarray:
    """Matrix-side group starts of every level, flattened: entry 2^l - 2 + q is where
    the l-bit prefix q starts in matrix level l, 1 <= l < width (wt2wm.py:55-78)."""
    width = code_width(sigma)
    full = 1 << width
    src = np.asarray(counts, dtype=np.int64)
    if src.size > full:
        raise ValueError("histogram longer than the code range")
    c = np.zeros(full, dtype=np.int64)
    c[: src.size] = src
    table = np.zeros(max(full - 2, 0), dtype=np.int64)
    if width >= 2:
        chain = _fold_chain(c, width)
        for ell in range(1, width):
            h = chain[ell]
            order = bit_reversal_permutation(ell)  # matrix rank r holds prefix order[r]
            starts = np.zeros(1 << ell, dtype=np.int64)
            starts[order] = np.cumsum(h[order]) - h[order]
            table[(1 << ell) - 2 : (2 << ell) - 2] = starts
    return table


class TreeToMatrixMap:
    """Constant-time map of tree level positions to matrix positions (wt2wm.py:81-134),
    from the histogram only: the unary histogram code with a rank/select
    directory (built on the GPU) and the flat start table."""

    def __init__(self, counts, sigma: int):
        from .bitvec import RankSelectBitVector

        if sigma < 1:
            raise ValueError("alphabet size must be at least 1")
        c = np.asarray(counts, dtype=np.int64)
        if c.size > (1 << code_width(sigma)):
            raise ValueError("histogram longer than the code range")
        if c.size > sigma and int(c[sigma:].max(initial=0)) > 0:
            raise ValueError("counts above the alphabet bound must be zero")
        if c.size and int(c.min()) < 0:
            raise ValueError("counts must be nonnegative")
        head = np.zeros(sigma, dtype=np.int64)
        head[: min(c.size, sigma)] = c[:sigma]
        self.sigma = sigma
        self.width = code_width(sigma)
        self.n = int(head.sum())
        self.unary = RankSelectBitVector(unary_histogram(head))
        self.starts = interval_start_table(head, sigma)

    def map_position(self, level: int, i: int) -> int:
        if not 0 <= level < self.width:
            raise IndexError(f"level {level} out of range for width {self.width}")
        if not 0 <= i < self.n:
            raise IndexError(f"position {i} out of range for length {self.n}")
        if level <= 1:
            return i
        u = self.unary
        # the (i+1)-th smallest symbol shares its level-bit prefix with the one at tree position i
        value = u.rank(0, u.select(1, i + 1))
        shift = self.width - level
        prefix = value >> shift
        # tree start of the prefix group = symbols smaller than prefix << shift
        first = 0 if prefix == 0 else u.rank(1, u.select(0, prefix << shift))
        return int(self.starts[(1 << level) - 2 + prefix]) + (i - first)


def recover_histogram(wt: LevelWiseWaveletTree) -> np.ndarray:
    """Histogram from the tree alone (wt2wm.py:137-156): split [0, n) level by level,
    a group's zero count being its left child's size.  One batch of device rank
    queries per level."""
    torch = _torch()
    from .support import DeviceSupport

    if wt.width == 0:
        return np.array([wt.n], dtype=np.int64)
    sup = DeviceSupport.from_structure(wt)
    bounds = np.array([0, wt.n], dtype=np.int64)
    for ell in range(wt.width):
        r1 = sup.level_rank1(ell, torch.from_numpy(bounds)).cpu().numpy()
        z = bounds - r1  # zeros before each bound
        splits = bounds[:-1] + (z[1:] - z[:-1])
        merged = np.empty(2 * bounds.size - 1, dtype=np.int64)
        merged[0::2] = bounds
        merged[1::2] = splits
        bounds = merged
    return np.diff(bounds)


def _level_plans(counts: np.ndarray, width: int):
    """Per level l >= 2: (bounds, source starts) of the gather_bits plan that moves
    the tree's prefix groups into bit-reversed order (wt2wm.py:205-225)."""
    chain = _fold_chain(counts, width)
    plans = {}
    for ell in range(2, width):
        h = chain[ell]
        order = bit_reversal_permutation(ell)
        tree_start = np.cumsum(h) - h
        lens = h[order]
        keep = lens > 0
        lens = lens[keep]
        src = tree_start[order][keep]
        bounds = np.zeros(lens.size + 1, dtype=np.int64)
        np.cumsum(lens, out=bounds[1:])
        plans[ell] = (bounds, np.ascontiguousarray(src, dtype=np.int64))
    return chain, plans


class ConversionPlan:
    """Device-resident gather_bits plans of every level >= 2 (one H2D copy)."""

    def __init__(self, counts, n: int, sigma: int, device):
        torch = _torch()
        self.n, self.sigma, self.width = int(n), int(sigma), code_width(sigma)
        chain, plans = _level_plans(np.asarray(counts, dtype=np.int64), self.width)
        self.zeros = [int(zeros_from_histogram(chain[ell + 1])) for ell in range(self.width)]
        parts, self.slices = [], {}
        off = 0
        for ell, (bounds, src) in plans.items():
            self.slices[ell] = (off, bounds.size, off + bounds.size, src.size)
            parts += [bounds, src]
            off += bounds.size + src.size
        flat = np.concatenate(parts) if parts else np.zeros(1, dtype=np.int64)
        host = torch.from_numpy(flat).pin_memory() if torch.cuda.is_available() else torch.from_numpy(flat)
        self.buf = host.to(device, non_blocking=True)

    def run(self, tree_words, out, builder):
        nwords = (self.n + 63) >> 6
        for ell in range(min(self.width, 2)):
            out[ell].copy_(tree_words[ell])
        if self.n == 0:
            return out
        for ell, (b0, nb, s0, ns) in self.slices.items():
            builder.merge_bits(out[ell], 0, nwords, self.n, self.buf[b0 : b0 + nb], self.buf[s0 : s0 + ns],
                               tree_words[ell], dst_offset_words=0)
        return out


def convert_levels_device(tree_words, n: int, sigma: int, counts, builder=None, plan=None):
    """Device conversion core: int64 tensor [width, ceil(n/64)] of tree level words
    -> (matrix level words tensor, zero counts).  Levels >= 2 go through
    wvlt_merge_bits; levels 0 and 1 are copied."""
    torch = _torch()
    from .device import default_builder

    b = builder or default_builder(tree_words.device)
    plan = plan or ConversionPlan(counts, n, sigma, tree_words.device)
    out = torch.empty_like(tree_words)
    plan.run(tree_words, out, b)
    return out, list(plan.zeros)


def convert_wt_to_wm(wt: LevelWiseWaveletTree, text=None, histogram=None) -> WaveletMatrix:
    """Matrix equivalent of a tree without revisiting the text (wt2wm.py:159-227).

    The histogram comes from `histogram` if given, else from `text`, else it is
    recovered from the tree; the level reordering runs on the GPU."""
    torch = _torch()
    if not isinstance(wt, LevelWiseWaveletTree):
        raise TypeError("conversion starts from a wavelet tree")
    n, sigma, width = wt.n, wt.sigma, wt.width
    full = 1 << width
    if histogram is not None:
        h = np.asarray(histogram, dtype=np.int64)
        if h.size > full:
            raise ValueError("histogram longer than the code range")
        if h.size and int(h.min()) < 0:
            raise ValueError("counts must be nonnegative")
        counts = np.zeros(full, dtype=np.int64)
        counts[: h.size] = h
        if int(counts.sum()) != n:
            raise ValueError("histogram total disagrees with the structure length")
        if int(counts[sigma:].max(initial=0)) > 0:
            raise ValueError("counts above the alphabet bound must be zero")
    elif text is not None:
        arr = np.asarray(text)
        if arr.size != n:
            raise ValueError("text length disagrees with the structure")
        counts = _histogram(arr, sigma, full)
    else:
        counts = recover_histogram(wt)
    if width == 0:
        return WaveletMatrix(n, sigma, [], [])
    nwords = (n + 63) >> 6
    host = np.zeros((width, nwords), dtype=np.uint64)
    for ell, vec in enumerate(wt.levels):
        host[ell] = vec.words
    dev_words = torch.from_numpy(host.view(np.int64)).cuda()
    out, zeros = convert_levels_device(dev_words, n, sigma, counts)
    words = out.cpu().numpy().view(np.uint64)
    levels = [BitVector(n, words[ell].copy()) for ell in range(width)]
    return WaveletMatrix(n, sigma, levels, zeros)


def _histogram(arr: np.ndarray, sigma: int, full: int) -> np.ndarray:
    """Device histogram of a host text (wvlt_histogram); ValueError on symbols outside [0, sigma)."""
    torch = _torch()
    from . import _lib
    from .construct import _device_text

    counts = np.zeros(full, dtype=np.int64)
    if arr.size == 0:
        return counts
    if arr.ndim != 1 or not np.issubdtype(arr.dtype, np.integer):
        raise ValueError("text must be a one-dimensional integer array")
    if int(arr.min()) < 0 or int(arr.max()) >= sigma:
        raise ValueError(f"symbols must lie in [0, {sigma})")
    dev = torch.from_numpy(_device_text(np.ascontiguousarray(arr), sigma)).cuda()
    hist = torch.zeros(full, dtype=torch.int64, device=dev.device)
    status = torch.zeros(1, dtype=torch.int32, device=dev.device)
    lib = _lib.load()
    rc = lib.wvlt_histogram(dev.data_ptr(), dev.element_size(), int(dev.numel()), int(sigma), hist.data_ptr(),
                            status.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    return hist.cpu().numpy()
