"""Build the in-tree CUDA library (sm_100a) with plain nvcc.

The shared object lands next to this file as ``_wvlt_b200.so`` so it travels
with the repository snapshot to the GPU box (it is git-ignored, not
gpurun-ignored).  No JIT cache is involved.

The product library is always built with exactly ``NVCC_FLAGS`` (nothing is
read from the environment).  A sidecar stamp holds the SHA-256 of the flags and
of every source byte, so a library built from other sources or flags (or copied
over the product file) is rebuilt.  Tuning experiments go through
``build_variant``, which writes to ``tools/variants/<name>.so`` and never
touches the product library.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
INCLUDE = REPO_DIR / "include"
LIB_NAME = "_wvlt_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME

SOURCES = [CSRC / "wvlt_b200.cu"]
INCLUDED = [CSRC / "support.cuh", CSRC / "k8.cuh", CSRC / "k8q.cuh", CSRC / "k16.cuh", CSRC / "k16q.cuh", CSRC / "k32.cuh"]  # #included by wvlt_b200.cu
HEADERS = [INCLUDE / "wvlt_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
]
STAMP_PATH = PKG_DIR / (LIB_NAME + ".stamp")
VARIANT_DIR = REPO_DIR / "tools" / "variants"


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build the extension")


def source_digest(flags=NVCC_FLAGS) -> str:
    h = hashlib.sha256()
    h.update("\0".join(flags).encode())
    for src in SOURCES + INCLUDED + HEADERS:
        h.update(src.name.encode())
        h.update(src.read_bytes())
    return h.hexdigest()


def _lib_digest() -> str:
    return hashlib.sha256(LIB_PATH.read_bytes()).hexdigest()


def is_stale() -> bool:
    """True unless the library exists and the stamp matches both the current
    sources + flags and the library file itself."""
    if not LIB_PATH.exists() or not STAMP_PATH.exists():
        return True
    try:
        src_digest, lib_digest = STAMP_PATH.read_text().split()
    except ValueError:
        return True
    return src_digest != source_digest() or lib_digest != _lib_digest()


def _nvcc(flags, out: Path, verbose: bool) -> None:
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc_path(), *flags, f"-I{INCLUDE}", *map(str, SOURCES), "-o", str(tmp), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG_DIR / "csrc" / "build.log"
    log.write_text(" ".join(cmd) + "\n\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc failed (exit {res.returncode}); see {log}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not is_stale():
        return LIB_PATH
    _nvcc(NVCC_FLAGS, LIB_PATH, verbose)
    STAMP_PATH.write_text(f"{source_digest()} {_lib_digest()}\n")
    return LIB_PATH


def build_variant(name: str, defines, verbose: bool = False) -> Path:
    """A tuning variant (extra ``-D`` defines) at tools/variants/<name>.so, for
    experiments only; load it with ``_lib.load_variant``."""
    VARIANT_DIR.mkdir(parents=True, exist_ok=True)
    out = VARIANT_DIR / f"{name}.so"
    _nvcc([*NVCC_FLAGS, *(f"-D{d}" for d in defines)], out, verbose)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
