"""Device-resident construction through the C ABI (include/wvlt_b200.h).

PyTorch is used only for plumbing: device buffers (caching allocator), the
current CUDA stream and host<->device copies.  All arithmetic runs in the
hand-written sm_100a kernels of ``csrc/wvlt_b200.cu``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bitperm import code_width

_TORCH = None


def _torch():
    global _TORCH
    if _TORCH is None:
        import torch

        _TORCH = torch
    return _TORCH


def sym_dtype_for_sigma(sigma: int):
    """Narrowest unsigned storage for symbols of [0, sigma) (cli._min_dtype, cli.py:59-66)."""
    if sigma <= 1 << 8:
        return np.uint8
    if sigma <= 1 << 16:
        return np.uint16
    return np.uint32


_TORCH_SYM = {1: "uint8", 2: "uint16", 4: "uint32"}


@dataclass
class DeviceBuild:
    """One device-resident build.  Tensors live on the build's device."""

    kind: str
    n: int
    sigma: int
    width: int
    level_words: object  # torch.int64 [width, ceil(n/64)] (bit pattern = uint64 words)
    zeros: object        # torch.int64 [width]
    hist: object         # torch.int64 [2^width]
    borders: object      # torch.int64 [2^width - 2] or None
    status: object = None  # torch.int32 [1]: WVLT_STATUS_RANGE bit set on a bad symbol

    def to_host(self):
        """(level_words uint64 ndarray, zeros list, hist ndarray) after a device->host copy."""
        lw = self.level_words.cpu().numpy().view(np.uint64)
        zeros = [int(z) for z in self.zeros.cpu().tolist()] if self.width else []
        return lw, zeros, (self.hist.cpu().numpy() if self.hist is not None else None)


# texts at least this long are copied to aligned memory when their pointer is not 16-byte
# aligned (shorter ones keep the kernels' element-wise paths, which the tests exercise)
REALIGN_MIN = 1 << 22


class DeviceBuilder:
    """Builds wavelet trees / matrices on one CUDA device, reusing a workspace."""

    def __init__(self, device=None):
        torch = _torch()
        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("the wavelet construction path needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self._ws = {}  # stream handle -> workspace (builds on different streams never share one)

    # -- buffers -------------------------------------------------------------
    def workspace_bytes(self, n: int, sym_bytes: int, sigma: int, kind: str) -> int:
        need = int(self.lib.wvlt_workspace_bytes(int(n), int(sym_bytes), int(sigma), _lib.KINDS[kind]))
        if need == 0 and code_width(sigma) > _lib.MAX_WIDTH:
            raise ValueError(f"alphabet size {sigma} exceeds the supported code width {_lib.MAX_WIDTH}")
        return need

    def workspace(self, n: int, sym_bytes: int, sigma: int, kind: str, stream=None):
        """The workspace of builds on ``stream`` (default: the current stream), grown
        on demand.  It is allocated on that stream, so the caching allocator only
        recycles a replaced one after the stream's queued work."""
        torch = _torch()
        need = self.workspace_bytes(n, sym_bytes, sigma, kind)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        ws = self._ws.get(s.cuda_stream)
        if ws is None or ws.numel() < need:
            with torch.cuda.stream(s):
                ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
            self._ws[s.cuda_stream] = ws
        return ws, need

    def alloc_outputs(self, n: int, sigma: int, borders: bool = False):
        torch = _torch()
        w = code_width(sigma)
        nwords = (n + 63) >> 6
        lw = torch.empty((w, nwords), dtype=torch.int64, device=self.device)
        zeros = torch.empty(max(w, 1), dtype=torch.int64, device=self.device)[:w]
        hist = torch.empty(1 << w, dtype=torch.int64, device=self.device)
        bd = torch.empty(max((1 << w) - 2, 1), dtype=torch.int64, device=self.device) if borders and w >= 2 else None
        status = torch.empty(1, dtype=torch.int32, device=self.device)
        return lw, zeros, hist, bd, status

    # -- builds --------------------------------------------------------------
    def build(self, text, sigma: int, kind: str = "wm", *, borders: bool = False, histogram: bool = False,
              outputs=None, stream=None, check: bool = True, workspace=None) -> DeviceBuild:
        """Build from a device tensor of uint8/uint16/uint32 symbols in [0, sigma).

        ``outputs`` may pass preallocated (level_words, zeros, hist, borders, status)
        from ``alloc_outputs`` (the benchmark does, to time the build alone).
        ``histogram`` also returns the symbol histogram; a WM build without
        histogram or borders skips the histogram kernel altogether (its tables
        come from the per-pass tile counts).
        With ``check`` the range status is read back (one device->host sync) and
        a bad symbol raises ValueError like construct._validated (construct.py:183-187).
        ``workspace`` passes a private uint8 device buffer instead of the per-stream
        shared one (a captured graph owns its own, see ``capture``).
        """
        torch = _torch()
        if kind not in _lib.KINDS:
            raise ValueError(f"unknown structure kind {kind!r}")
        if text.device.type != "cuda":
            raise ValueError("DeviceBuilder.build expects a CUDA tensor")
        if text.dim() != 1:
            raise ValueError("text must be one-dimensional")
        sb = text.element_size()
        if text.dtype not in (torch.uint8, torch.uint16, torch.uint32) or sb not in (1, 2, 4):
            raise ValueError("device text must be uint8, uint16 or uint32")
        if not text.is_contiguous():
            text = text.contiguous()
        sigma = int(sigma)
        if sigma < 1:
            raise ValueError("alphabet size must be at least 1")
        n = int(text.numel())
        w = code_width(sigma)
        if w > _lib.MAX_WIDTH:
            raise ValueError(f"alphabet size {sigma} exceeds the supported code width {_lib.MAX_WIDTH}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if n >= REALIGN_MIN and text.data_ptr() % 16:
            # a large text that does not start on a 16-byte boundary (a slice at an odd
            # offset): the kernels would take their element-wise loads (c3: 5.2 ms
            # instead of 0.64 ms), one device copy into aligned memory costs 2 n bytes
            with torch.cuda.stream(s):
                text = text.clone()
        if outputs is None:
            with torch.cuda.stream(s):
                outputs = self.alloc_outputs(n, sigma, borders)
        lw, zeros, hist, bd, status = outputs
        if workspace is None:
            ws, need = self.workspace(n, sb, sigma, kind, s)
        else:
            ws, need = workspace, self.workspace_bytes(n, sb, sigma, kind)
            if ws.numel() < need:
                raise ValueError(f"workspace holds {ws.numel()} bytes, the build needs {need}")
        rc = self.lib.wvlt_build_device(
            text.data_ptr() if n else None, sb, n, sigma, _lib.KINDS[kind],
            lw.data_ptr() if lw.numel() else None, zeros.data_ptr() if w else None,
            hist.data_ptr() if histogram else None,
            bd.data_ptr() if bd is not None else None, ws.data_ptr(), need, status.data_ptr(), s.cuda_stream)
        _lib.check(rc)
        if check and int(status.item()) & _lib.STATUS_RANGE:
            raise ValueError(f"symbols must lie in [0, {sigma})")
        return DeviceBuild(kind, n, sigma, w, lw, zeros, hist if histogram else None, bd, status)

    def capture(self, text, sigma: int, kind: str = "wm", *, histogram: bool = False,
                borders: bool = False) -> "BuildGraph":
        """Capture one build of ``text`` (a device tensor kept as the graph's input
        buffer) into a CUDA graph: small, launch-bound builds replay it with one
        launch.  Refill ``text`` in place and call ``replay()`` for the next build
        of the same length / alphabet / kind.

        The graph bakes in the workspace address, so it gets a private workspace
        that the returned BuildGraph keeps alive (never the per-stream shared one,
        which a later build could replace and free under the graph)."""
        torch = _torch()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        n = int(text.numel())
        need = self.workspace_bytes(n, text.element_size(), sigma, kind)
        with torch.cuda.stream(s):
            outputs = self.alloc_outputs(n, sigma, borders)
            ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
            self.build(text, sigma, kind, histogram=histogram, borders=borders, outputs=outputs, stream=s,
                       check=False, workspace=ws)  # warm-up
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            res = self.build(text, sigma, kind, histogram=histogram, borders=borders, outputs=outputs,
                             stream=torch.cuda.current_stream(self.device), check=False, workspace=ws)
        return BuildGraph(g, res, text, ws)

    def build_host(self, arr: np.ndarray, sigma: int, kind: str, *, out_words: np.ndarray | None = None,
                   histogram: bool = False, stream=None):
        """Host buffers in and out through wvlt_build_host (H2D, build, D2H, sync).

        ``arr`` is a contiguous uint8/uint16/uint32 host array (page-locked for
        full PCIe bandwidth).  Returns (level_words uint64[w, ceil(n/64)], zeros,
        hist or None).
        """
        words, zeros, hist, _ = self.build_host_ex(arr, sigma, kind, out_words=out_words, histogram=histogram,
                                                   borders=False, stream=stream)
        return words, zeros, hist

    def build_host_ex(self, arr: np.ndarray, sigma: int, kind: str, *, out_words: np.ndarray | None = None,
                      histogram: bool = False, borders: bool = False, stream=None):
        """``build_host`` that can also return the node borders (wvlt_build_host_borders):
        (level_words, zeros, hist or None, borders int64[2^w - 2] or None)."""
        torch = _torch()
        if arr.dtype not in (np.uint8, np.uint16, np.uint32) or not arr.flags.c_contiguous:
            raise ValueError("host text must be a contiguous uint8/uint16/uint32 array")
        n = int(arr.size)
        sb = arr.dtype.itemsize
        w = code_width(sigma)
        nwords = (n + 63) >> 6
        if out_words is None:
            out_words = np.empty((w, nwords), dtype=np.uint64)
        zeros = np.zeros(max(w, 1), dtype=np.int64)
        hist = np.zeros(1 << w, dtype=np.int64)
        bd = np.zeros(max((1 << w) - 2, 1), dtype=np.int64)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            dev_text = torch.empty(max(n * sb, 16), dtype=torch.uint8, device=self.device)
            dev_words = torch.empty(max(w * nwords, 1), dtype=torch.int64, device=self.device)
            dev_small = torch.empty((2 << w) + w + 1, dtype=torch.int64, device=self.device)
        ws, need = self.workspace(n, sb, sigma, kind, s)
        rc = self.lib.wvlt_build_host_borders(
            arr.ctypes.data if n else None, sb, n, sigma, _lib.KINDS[kind],
            out_words.ctypes.data if out_words.size else None, zeros.ctypes.data,
            hist.ctypes.data if histogram else None, bd.ctypes.data if borders else None,
            dev_text.data_ptr(), dev_words.data_ptr(), dev_small.data_ptr(), ws.data_ptr(), need, s.cuda_stream)
        if rc == _lib.E_RANGE:
            raise ValueError(f"symbols must lie in [0, {sigma})")
        _lib.check(rc)
        return (out_words, [int(z) for z in zeros[:w]], (hist if histogram else None),
                (bd[: max((1 << w) - 2, 0)] if borders else None))

    def build_host_batch(self, arrs, sigma: int, kind: str, *, out_words=None, histogram: bool = False,
                         stream=None):
        """A queue of independent builds through wvlt_build_host_batch: the upload of
        text i+1, the build of text i and the download of build i-1's levels overlap
        (three streams, double-buffered device buffers).

        ``arrs`` are contiguous host arrays of one dtype (page-locked for full PCIe
        bandwidth); ``out_words[i]`` (optional) receives build i's level words.
        Returns a list of (level_words, zeros, hist or None) per text, like
        build_host.  Raises ValueError if any text has a symbol outside [0, sigma).
        """
        torch = _torch()
        arrs = list(arrs)
        count = len(arrs)
        if count == 0:
            return []
        dt = arrs[0].dtype
        if dt not in (np.uint8, np.uint16, np.uint32):
            raise ValueError("host texts must be contiguous uint8/uint16/uint32 arrays")
        for a in arrs:
            if a.dtype != dt or not a.flags.c_contiguous or a.ndim != 1:
                raise ValueError("host texts must be contiguous 1-D arrays of one dtype")
        sb = dt.itemsize
        w = code_width(sigma)
        ns = np.array([a.size for a in arrs], dtype=np.int64)
        nmax = int(ns.max())
        nw = [(int(n) + 63) >> 6 for n in ns]
        if out_words is None:
            out_words = [np.empty((w, k), dtype=np.uint64) for k in nw]
        for o, k in zip(out_words, nw):
            if o.dtype != np.uint64 or not o.flags.c_contiguous or o.size < w * k:
                raise ValueError("out_words[i] must be a contiguous uint64 array of width x ceil(n_i/64) words")
        zeros = np.zeros((count, max(w, 1)), dtype=np.int64)
        hist = np.zeros((count, 1 << w), dtype=np.int64) if histogram else None
        status = np.zeros(count, dtype=np.int32)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        text_slot = max(nmax * sb, 16)
        text_slot = (text_slot + 255) // 256 * 256
        words_slot = max(w * ((nmax + 63) >> 6) * 8, 8)
        words_slot = (words_slot + 255) // 256 * 256
        with torch.cuda.stream(s):
            dev_text = torch.empty(2 * text_slot, dtype=torch.uint8, device=self.device)
            dev_words = torch.empty(2 * words_slot // 8, dtype=torch.int64, device=self.device)
            dev_small = torch.empty(2 * ((1 << w) + w + 1), dtype=torch.int64, device=self.device)
        ws, need = self.workspace(nmax, sb, sigma, kind, s)
        texts_p = (ctypes.c_void_p * count)(*[a.ctypes.data if a.size else None for a in arrs])
        words_p = (ctypes.c_void_p * count)(*[o.ctypes.data if o.size else None for o in out_words])
        rc = self.lib.wvlt_build_host_batch(
            count, ctypes.cast(texts_p, ctypes.c_void_p), ns.ctypes.data, sb, sigma, _lib.KINDS[kind],
            ctypes.cast(words_p, ctypes.c_void_p), zeros.ctypes.data, hist.ctypes.data if histogram else None,
            status.ctypes.data, dev_text.data_ptr(), text_slot, dev_words.data_ptr(), words_slot,
            dev_small.data_ptr(), ws.data_ptr(), need, s.cuda_stream)
        if rc == _lib.E_RANGE:
            bad = [i for i in range(count) if status[i]]
            raise ValueError(f"symbols must lie in [0, {sigma}) (texts {bad})")
        _lib.check(rc)
        return [(out_words[i], [int(z) for z in zeros[i, :w]], (hist[i] if histogram else None))
                for i in range(count)]

    def merge_bits(self, dst_words, word_lo: int, word_hi: int, n_bits: int, bounds, src_starts, src_words,
                   stream=None, dst_offset_words: int = 0) -> None:
        """gather_bits (_kernels.py:196-232) on device tensors (int64 views of uint64 words).

        Destination word ``wd`` of [word_lo, word_hi) is written at
        ``dst_words[wd - dst_offset_words]`` (so a buffer holding just the owned
        range can be passed with ``dst_offset_words = word_lo``).
        """
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        ntasks = int(bounds.numel()) - 1
        rc = self.lib.wvlt_merge_bits(dst_words.data_ptr() - 8 * int(dst_offset_words), int(word_lo), int(word_hi),
                                      int(n_bits),
                                      bounds.data_ptr() if ntasks > 0 else None,
                                      src_starts.data_ptr() if ntasks > 0 else None, max(ntasks, 0),
                                      src_words.data_ptr() if src_words.numel() else None, s.cuda_stream)
        _lib.check(rc)


class BuildGraph:
    """A captured build (DeviceBuilder.capture): ``replay()`` reruns it on the current
    contents of ``text``; ``result`` holds the output tensors, ``check()`` raises
    ValueError if the last replay saw a symbol outside [0, sigma)."""

    def __init__(self, graph, result: DeviceBuild, text, workspace):
        self.graph, self.result, self.text = graph, result, text
        self.workspace = workspace  # the address the graph writes into: owned here

    def replay(self) -> DeviceBuild:
        self.graph.replay()
        return self.result

    def check(self) -> None:
        if int(self.result.status.item()) & _lib.STATUS_RANGE:
            raise ValueError(f"symbols must lie in [0, {self.result.sigma})")


_BUILDERS: dict = {}


def default_builder(device=None) -> DeviceBuilder:
    torch = _torch()
    key = str(device) if device is not None else f"cuda:{torch.cuda.current_device()}" if torch.cuda.is_available() else "cuda"
    b = _BUILDERS.get(key)
    if b is None:
        b = DeviceBuilder(device)
        _BUILDERS[key] = b
    return b
