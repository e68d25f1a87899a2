"""ctypes binding of the in-tree CUDA library (include/wvlt_b200.h).

There is no fallback: if the shared object is missing or cannot be loaded
this raises, and every build entry point raises with it.
"""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_wvlt_b200.so"
HEADER = _PKG.parent / "include" / "wvlt_b200.h"

KIND_WT = 0
KIND_WM = 1
KINDS = {"wt": KIND_WT, "wm": KIND_WM}
E_ARG, E_WIDTH, E_WORKSPACE, E_RANGE = -1, -2, -3, -4
STATUS_RANGE = 1
MAX_WIDTH = 28
STAGE_MEMSET, STAGE_HIST, STAGE_TABLES, STAGE_PASS0, STAGE_SCAN0, STAGE_REORDER = 0, 1, 2, 3, 64, 60

_lib = None


class WvltError(RuntimeError):
    """A CUDA or contract error reported by the C ABI."""


def load():
    """Load the library; raises if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a); the wavelet construction path has no CPU fallback"
        )
    _lib = _bind(ctypes.CDLL(str(LIB_PATH)))
    return _lib


def load_variant(path) -> ctypes.CDLL:
    """Experiments only (tools/variant_bench.py): bind a tuning variant built by
    ``_build.build_variant`` in place of the product library for this process.
    Must be called before anything else loads the library."""
    global _lib
    path = Path(path).resolve()
    if path.parent != (_PKG.parent / "tools" / "variants").resolve():
        raise ValueError("variants live in tools/variants/")
    if _lib is not None:
        raise RuntimeError("the product library is already loaded in this process")
    _lib = _bind(ctypes.CDLL(str(path)))
    return _lib


def _bind(L):
    i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
    L.wvlt_abi_version.argtypes = []
    L.wvlt_abi_version.restype = i32
    L.wvlt_error_string.argtypes = [i32]
    L.wvlt_error_string.restype = ctypes.c_char_p
    L.wvlt_code_width.argtypes = [i64]
    L.wvlt_code_width.restype = i32
    L.wvlt_workspace_bytes.argtypes = [i64, i32, i64, i32]
    L.wvlt_workspace_bytes.restype = sz
    L.wvlt_workspace_parts.argtypes = [i64, i32, i64, i32, i32, i32, vp]
    L.wvlt_workspace_parts.restype = i32
    L.wvlt_histogram.argtypes = [vp, i32, i64, i64, vp, vp, vp]
    L.wvlt_histogram.restype = i32
    L.wvlt_build_device.argtypes = [vp, i32, i64, i64, i32, vp, vp, vp, vp, vp, sz, vp, vp]
    L.wvlt_build_device.restype = i32
    L.wvlt_build_host.argtypes = [vp, i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.wvlt_build_host.restype = i32
    L.wvlt_build_host_borders.argtypes = [vp, i32, i64, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.wvlt_build_host_borders.restype = i32
    L.wvlt_build_host_batch.argtypes = [i32, vp, vp, i32, i64, i32, vp, vp, vp, vp, vp, sz, vp, sz, vp, vp, sz, vp]
    L.wvlt_build_host_batch.restype = i32
    L.wvlt_merge_bits.argtypes = [vp, i64, i64, i64, vp, vp, i64, vp, vp]
    L.wvlt_merge_bits.restype = i32
    L.wvlt_merge_levels_peer.argtypes = [vp, i64, i32, i64, i64, i64, vp, vp, vp, vp, vp, vp, i32, vp]
    L.wvlt_merge_levels_peer.restype = i32
    L.wvlt_peer_plan.argtypes = [vp, i64, i64, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]
    L.wvlt_peer_plan.restype = i32
    L.wvlt_last_launches.argtypes = []
    L.wvlt_last_launches.restype = i32
    L.wvlt_rank_select_workspace_bytes.argtypes = [i64, i64]
    L.wvlt_rank_select_workspace_bytes.restype = sz
    L.wvlt_rank_select_build.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp, vp, sz, vp]
    L.wvlt_rank_select_build.restype = i32
    L.wvlt_query.argtypes = [i32, i32, vp, i64, i32, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, i64, vp]
    L.wvlt_query.restype = i32
    L.wvlt_profile_enable.argtypes = [i32]
    L.wvlt_profile_enable.restype = i32
    L.wvlt_profile_read.argtypes = [vp, vp, i32]
    L.wvlt_profile_read.restype = i32
    if L.wvlt_abi_version() != 1:
        raise ImportError("wvlt_b200 ABI version mismatch")
    return L


def workspace_parts(n: int, sym_bytes: int, sigma: int, kind: str, histogram: bool, borders: bool):
    """(positions, symbols, partial_bits) bytes of one build's workspace (wvlt_workspace_parts)."""
    out = (ctypes.c_size_t * 3)()
    rc = load().wvlt_workspace_parts(int(n), int(sym_bytes), int(sigma), KINDS[kind], int(histogram), int(borders), out)
    check(rc)
    return int(out[0]), int(out[1]), int(out[2])


def check(rc: int) -> None:
    if rc:
        msg = load().wvlt_error_string(rc).decode()
        raise WvltError(f"{msg} (code {rc})")


def profile_enable(on: bool) -> None:
    load().wvlt_profile_enable(1 if on else 0)


def profile_read(max_stages: int = 40) -> list[tuple[str, float]]:
    """[(stage name, ms)] of the last profiled wvlt_build_device on this thread."""
    ms = (ctypes.c_float * max_stages)()
    ids = (ctypes.c_int * max_stages)()
    k = load().wvlt_profile_read(ms, ids, max_stages)
    if k < 0:
        raise WvltError(f"profile read failed ({k})")
    names = {STAGE_MEMSET: "memset", STAGE_HIST: "hist", STAGE_TABLES: "tables", STAGE_REORDER: "reorder"}
    def name(i):
        if i in names:
            return names[i]
        return f"scan{i - STAGE_SCAN0}" if i >= STAGE_SCAN0 else f"pass{i - STAGE_PASS0}"

    return [(name(ids[i]), float(ms[i])) for i in range(k)]


def declared_symbols() -> list[str]:
    """Function names declared in include/wvlt_b200.h (the ABI contract)."""
    text = HEADER.read_text()
    return re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(wvlt_[a-z0-9_]+)\s*\(", text, re.M)
