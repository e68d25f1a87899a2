"""Rank/select view of a bit vector (mirror of the reference's bitvec.py:118-263).

`RankSelectBitVector(bits)` keeps the reference's attributes and semantics --
`rank(x, i)` counts bit x in [0, i), `select(x, j)` is the position of the
j-th (1-based) occurrence and raises AbsentOccurrenceError past the count --
but its directory (superblock / block zero counts and select samples) is built
by the GPU kernel `wvlt_rank_select_build`.  Single queries are then answered
on the host from that directory; batches go through support.DeviceSupport.
"""

from __future__ import annotations

import numpy as np

from .structures import BitVector
from .support import BLOCK_BITS, SELECT_SAMPLE, SUPERBLOCK_BITS, DeviceDirectory

WORD_BITS = 64
BLOCKS_PER_SUPER = SUPERBLOCK_BITS // BLOCK_BITS
WORDS_PER_BLOCK = BLOCK_BITS // WORD_BITS

__all__ = [
    "AbsentOccurrenceError", "BitVector", "RankSelectBitVector", "WORD_BITS", "SUPERBLOCK_BITS", "BLOCK_BITS",
    "BLOCKS_PER_SUPER", "WORDS_PER_BLOCK", "SELECT_SAMPLE",
]


class AbsentOccurrenceError(ValueError):
    """Select asked for an occurrence beyond the number present."""


def _popcount(word: int) -> int:
    return int(word).bit_count()


def _kth_set_bit(word: int, k: int) -> int:
    """0-based position of the k-th (1-based) set bit of a 64-bit word."""
    pos, width = 0, 64
    while width > 1:
        width >>= 1
        low = word & ((1 << width) - 1)
        c = _popcount(low)
        if k > c:
            k -= c
            word >>= width
            pos += width
        else:
            word = low
    return pos


class RankSelectBitVector:
    """Read-only rank/select view; directory built on the GPU."""

    __slots__ = ("bits", "_nblocks", "_nsuper", "_super_zeros", "_block_zeros", "_total_ones", "_total_zeros",
                 "_samples1", "_samples0")

    def __init__(self, bits: BitVector):
        self.bits = bits
        self._build()

    def _build(self) -> None:
        import torch

        n = self.bits.length
        self._nsuper = -(-n // SUPERBLOCK_BITS)
        self._nblocks = -(-n // BLOCK_BITS)
        if n == 0:
            self._super_zeros = np.zeros(0, dtype=np.int64)
            self._block_zeros = np.zeros(0, dtype=np.int64)
            self._samples1 = np.zeros(0, dtype=np.int64)
            self._samples0 = np.zeros(0, dtype=np.int64)
            self._total_ones = self._total_zeros = 0
            return
        words = torch.from_numpy(np.ascontiguousarray(self.bits.words).view(np.int64)).cuda()
        d = DeviceDirectory(words, 1, n).host_arrays(0)
        self._super_zeros = d["super_zeros"]
        self._block_zeros = d["block_zeros"]
        self._samples1 = d["samples1"]
        self._samples0 = d["samples0"]
        self._total_ones = int(d["ones"])
        self._total_zeros = n - self._total_ones

    def __len__(self) -> int:
        return self.bits.length

    def get(self, i: int) -> int:
        return self.bits.get(i)

    def count(self, x: int) -> int:
        return self._total_ones if x else self._total_zeros

    def rank(self, x: int, i: int) -> int:
        if x not in (0, 1):
            raise ValueError("bit value must be 0 or 1")
        if not 0 <= i <= self.bits.length:
            raise IndexError(f"rank position {i} outside [0, {self.bits.length}]")
        ones = self._ones_before(i)
        return ones if x else i - ones

    def _ones_before(self, i: int) -> int:
        if i == 0:
            return 0
        blk = min(i >> 8, self._nblocks - 1)
        r = (blk << 8) - int(self._super_zeros[blk >> 3]) - int(self._block_zeros[blk])
        words = self.bits.words
        last = i >> 6
        for w in range(blk << 2, last):
            r += _popcount(words[w])
        if i & 63:
            r += _popcount(int(words[last]) & ((1 << (i & 63)) - 1))
        return r

    def _before_superblock(self, x: int, s: int) -> int:
        if s >= self._nsuper:
            return self._total_ones if x else self._total_zeros
        z = int(self._super_zeros[s])
        return (s * SUPERBLOCK_BITS - z) if x else z

    def select(self, x: int, j: int) -> int:
        if x not in (0, 1):
            raise ValueError("bit value must be 0 or 1")
        if j < 1:
            raise ValueError("select ordinal is 1-based")
        if j > self.count(x):
            raise AbsentOccurrenceError(f"fewer than {j} occurrences of bit {x}")
        samples = self._samples1 if x else self._samples0
        k = (j - 1) // SELECT_SAMPLE
        lo = int(samples[k]) // SUPERBLOCK_BITS
        hi = int(samples[k + 1]) // SUPERBLOCK_BITS if k + 1 < samples.size else self._nsuper - 1
        while lo < hi:  # last superblock with fewer than j occurrences before it
            mid = (lo + hi + 1) // 2
            if self._before_superblock(x, mid) < j:
                lo = mid
            else:
                hi = mid - 1
        sz = int(self._super_zeros[lo])
        blk = lo * BLOCKS_PER_SUPER
        end = min(blk + BLOCKS_PER_SUPER, self._nblocks) - 1
        while blk < end:
            z = sz + int(self._block_zeros[blk + 1])
            if (((blk + 1) * BLOCK_BITS - z) if x else z) >= j:
                break
            blk += 1
        z = sz + int(self._block_zeros[blk])
        need = j - (((blk * BLOCK_BITS) - z) if x else z)
        n = self.bits.length
        words = self.bits.words
        w = blk * WORDS_PER_BLOCK
        while True:
            word = int(words[w])
            valid = min(64, n - w * 64)
            if not x:
                word = ~word & ((1 << valid) - 1)
            c = _popcount(word)
            if need <= c:
                return w * 64 + _kth_set_bit(word, need)
            need -= c
            w += 1

    def __repr__(self) -> str:
        return f"RankSelectBitVector({self.bits!r})"

