"""The C-ABI library loads on CPU and exports every symbol the header declares.
Only host-side functions are called (no CUDA work without a GPU)."""

from __future__ import annotations

import ctypes

from paper_1702_07578_b200 import _lib


def test_header_declares_the_abi():
    names = _lib.declared_symbols()
    for required in ("wvlt_abi_version", "wvlt_error_string", "wvlt_code_width", "wvlt_workspace_bytes",
                     "wvlt_histogram", "wvlt_build_device", "wvlt_build_host", "wvlt_merge_bits"):
        assert required in names


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    raw = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in _lib.declared_symbols():
        assert hasattr(raw, name), name
    assert L.wvlt_abi_version() == 1


def test_host_side_entry_points():
    L = _lib.load()
    for sigma in (0, 1, 2, 3, 5, 256, 257, 65536, 70000, 1 << 20):
        assert L.wvlt_code_width(sigma) == max(sigma - 1, 0).bit_length()
    assert L.wvlt_error_string(0) == b"ok"
    assert b"sigma" in L.wvlt_error_string(_lib.E_RANGE)
    assert L.wvlt_workspace_bytes(1 << 20, 1, 256, 1) > 0
    assert L.wvlt_workspace_bytes(1 << 20, 3, 256, 1) == 0       # bad symbol width
    assert L.wvlt_workspace_bytes(10, 4, 1 << 30, 0) == 0         # width above WVLT_MAX_WIDTH
    # workspace grows with n and carries two level-order buffers for multi-pass builds
    a = L.wvlt_workspace_bytes(1 << 20, 1, 256, 1)
    b = L.wvlt_workspace_bytes(1 << 21, 1, 256, 1)
    assert b > a


def test_device_entry_points_reject_bad_arguments_before_touching_the_device():
    L = _lib.load()
    assert L.wvlt_build_device(None, 3, 10, 4, 1, None, None, None, None, None, 0, None, None) == _lib.E_ARG
    assert L.wvlt_build_device(None, 1, 10, 4, 7, None, None, None, None, None, 0, None, None) == _lib.E_ARG
    assert L.wvlt_build_device(None, 1, 10, 1 << 30, 1, None, None, None, None, None, 0, None, None) == _lib.E_WIDTH
    assert L.wvlt_merge_bits(None, 5, 4, 10, None, None, 1, None, None) == _lib.E_ARG
