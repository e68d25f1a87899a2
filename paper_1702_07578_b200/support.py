"""Rank/select directories and batched queries on the device.

The directories are the reference's RankSelectBitVector arrays
(bitvec.py:118-163): zeros before every 2048-bit superblock, zeros before
every 256-bit block relative to its superblock, and the positions of every
8192nd one and zero.  `wvlt_rank_select_build` builds them for all levels of a
structure in two kernels and a scan; `wvlt_query` answers batches of
access / rank / select queries with the level walks of structures.py:107-256,
one thread per query.  No CPU fallback: a missing library or device raises.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .bitperm import code_width

SUPERBLOCK_BITS = 2048
BLOCK_BITS = 256
SELECT_SAMPLE = 8192

Q_ACCESS, Q_RANK, Q_SELECT, Q_BITRANK = 0, 1, 2, 3


def _torch():
    import torch

    return torch


def directory_shape(length: int) -> tuple[int, int, int, int]:
    """(words, superblocks, blocks, sample capacity) of one vector of `length` bits."""
    return ((length + 63) >> 6, -(-length // SUPERBLOCK_BITS), -(-length // BLOCK_BITS), -(-length // SELECT_SAMPLE))


class DeviceDirectory:
    """Directories of `nvec` equal-length bit vectors stored back to back on the device."""

    def __init__(self, words, nvec: int, length: int, stream=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("rank/select directories are built on the GPU (no CPU fallback)")
        lib = _lib.load()
        self.nvec, self.length = int(nvec), int(length)
        dev = words.device
        _, nsuper, nblocks, nsamp = directory_shape(self.length)
        i64 = dict(dtype=torch.int64, device=dev)
        self.super_zeros = torch.empty((self.nvec, max(nsuper, 1)), **i64)
        self.block_zeros = torch.empty((self.nvec, max(nblocks, 1)), **i64)
        self.samples1 = torch.empty((self.nvec, max(nsamp, 1)), **i64)
        self.samples0 = torch.empty((self.nvec, max(nsamp, 1)), **i64)
        self.ones = torch.zeros(max(self.nvec, 1), **i64)[: self.nvec]
        self.words = words
        if self.nvec == 0:
            return
        need = int(lib.wvlt_rank_select_workspace_bytes(self.nvec, self.length))
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        rc = lib.wvlt_rank_select_build(words.data_ptr() if words.numel() else None, self.nvec, self.length,
                                        self.super_zeros.data_ptr(), self.block_zeros.data_ptr(),
                                        self.samples1.data_ptr(), self.samples0.data_ptr(),
                                        self.ones.data_ptr() if self.nvec else None, ws.data_ptr(), need,
                                        s.cuda_stream)
        _lib.check(rc)
        self._ws = ws  # kept alive until the stream has consumed it

    def host_arrays(self, v: int) -> dict:
        """Vector v's directory as host arrays in the reference's shapes."""
        _, nsuper, nblocks, _ = directory_shape(self.length)
        ones = int(self.ones[v].item()) if self.nvec else 0
        zeros = self.length - ones
        n1 = -(-ones // SELECT_SAMPLE)
        n0 = -(-zeros // SELECT_SAMPLE)
        return {
            "super_zeros": self.super_zeros[v, :nsuper].cpu().numpy().copy(),
            "block_zeros": self.block_zeros[v, :nblocks].cpu().numpy().copy(),
            "samples1": self.samples1[v, :n1].cpu().numpy().copy(),
            "samples0": self.samples0[v, :n0].cpu().numpy().copy(),
            "ones": ones,
        }


class DeviceSupport:
    """A structure's levels on the device with their directories: batched queries.

    ``kind`` is "wt" or "wm"; ``level_words`` an int64 tensor [width, ceil(n/64)]
    (uint64 bit patterns, the build's layout); ``zeros`` the WM zero counts.
    """

    def __init__(self, kind: str, n: int, sigma: int, level_words, zeros=None, stream=None):
        torch = _torch()
        if kind not in ("wt", "wm"):
            raise ValueError(f"unknown structure kind {kind!r}")
        self.kind, self.n, self.sigma = kind, int(n), int(sigma)
        self.width = code_width(self.sigma)
        self.lib = _lib.load()
        dev = level_words.device
        self.device = dev
        self.words = level_words.contiguous()
        self.dir = DeviceDirectory(self.words, self.width, self.n, stream)
        if kind == "wm":
            z = torch.as_tensor(list(zeros) if zeros is not None else [0] * self.width, dtype=torch.int64)
            self.zeros = z.to(dev)
        else:
            self.zeros = None

    @classmethod
    def from_build(cls, build, stream=None):
        return cls(build.kind, build.n, build.sigma, build.level_words, build.zeros if build.kind == "wm" else None,
                   stream)

    @classmethod
    def from_structure(cls, st, device=None):
        torch = _torch()
        dev = torch.device("cuda") if device is None else torch.device(device)
        nw = (st.n + 63) >> 6
        host = np.zeros((st.width, nw), dtype=np.uint64)
        for ell, vec in enumerate(st.levels):
            host[ell] = vec.words
        words = torch.from_numpy(host.view(np.int64)).to(dev)
        return cls(st.kind, st.n, st.sigma, words, getattr(st, "zeros", None))

    # -- batched queries (structures.py:107-256 semantics, errors of _check_*) --
    def _run(self, op: int, sym, arg):
        torch = _torch()
        arg = torch.as_tensor(arg, dtype=torch.int64, device=self.device).contiguous()
        out = torch.empty_like(arg)
        sym_t = None
        sym_scalar = 0
        if sym is not None:
            if isinstance(sym, (int, np.integer)):
                sym_scalar = int(sym)
            else:
                sym_t = torch.as_tensor(sym, dtype=torch.int64, device=self.device).contiguous()
                if sym_t.shape != arg.shape:
                    raise ValueError("symbols and arguments must have the same shape")
        d = self.dir
        s = torch.cuda.current_stream(self.device)
        rc = self.lib.wvlt_query(
            1 if self.kind == "wm" else 0, op, self.words.data_ptr() if self.words.numel() else None, self.n,
            self.width, self.zeros.data_ptr() if self.zeros is not None and self.width else None,
            d.super_zeros.data_ptr(), d.block_zeros.data_ptr(), d.samples1.data_ptr(), d.samples0.data_ptr(),
            d.ones.data_ptr() if self.width else None, sym_t.data_ptr() if sym_t is not None else None,
            sym_scalar, arg.data_ptr(), out.data_ptr(), int(arg.numel()), s.cuda_stream)
        _lib.check(rc)
        return out

    def _check_symbols(self, c):
        torch = _torch()
        if isinstance(c, (int, np.integer)):
            if not 0 <= int(c) < self.sigma:
                raise ValueError(f"symbol {int(c)} outside alphabet [0, {self.sigma})")
        else:
            ct = torch.as_tensor(c)
            if ct.numel() and (int(ct.min()) < 0 or int(ct.max()) >= self.sigma):
                raise ValueError(f"symbol outside alphabet [0, {self.sigma})")

    def access(self, positions):
        torch = _torch()
        p = torch.as_tensor(positions, dtype=torch.int64, device=self.device)
        if p.numel() and (int(p.min()) < 0 or int(p.max()) >= self.n):
            raise IndexError(f"position out of range for length {self.n}")
        return self._run(Q_ACCESS, None, p)

    def rank(self, c, positions):
        torch = _torch()
        self._check_symbols(c)
        p = torch.as_tensor(positions, dtype=torch.int64, device=self.device)
        if p.numel() and (int(p.min()) < 0 or int(p.max()) > self.n):
            raise IndexError(f"rank prefix length out of range for length {self.n}")
        return self._run(Q_RANK, c, p)

    def level_rank1(self, level: int, positions):
        """Ones of one level in [0, p) for every p (the directory's rank1, batched)."""
        torch = _torch()
        if not 0 <= level < self.width:
            raise IndexError(f"level {level} out of range for width {self.width}")
        p = torch.as_tensor(positions, dtype=torch.int64, device=self.device)
        if p.numel() and (int(p.min()) < 0 or int(p.max()) > self.n):
            raise IndexError(f"rank position out of range for length {self.n}")
        return self._run(Q_BITRANK, int(level), p)

    def select(self, c, ordinals):
        """Positions of the j-th occurrences (1-based); -1 where fewer occurrences exist."""
        torch = _torch()
        self._check_symbols(c)
        j = torch.as_tensor(ordinals, dtype=torch.int64, device=self.device)
        if j.numel() and int(j.min()) < 1:
            raise ValueError("occurrence ordinals are 1-based")
        return self._run(Q_SELECT, c, j)
