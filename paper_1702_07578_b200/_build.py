"""Build the in-tree CUDA library (sm_100a) with plain nvcc.

The shared object lands next to this file as ``_wvlt_b200.so`` so it travels
with the repository snapshot to the GPU box (it is git-ignored, not
gpurun-ignored).  No JIT cache is involved.
"""

from __future__ import annotations

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
INCLUDED = [CSRC / "support.cuh", CSRC / "k8.cuh", CSRC / "k16.cuh", CSRC / "k32.cuh"]  # #included by wvlt_b200.cu
HEADERS = [INCLUDE / "wvlt_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
]
EXTRA_FLAGS = os.environ.get("WVLT_NVCC_EXTRA", "").split()


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build the extension")


def is_stale() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    return any(src.stat().st_mtime > built for src in SOURCES + INCLUDED + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not is_stale():
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc_path(), *NVCC_FLAGS, *EXTRA_FLAGS, f"-I{INCLUDE}", *map(str, SOURCES), "-o", str(tmp), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG_DIR / "csrc" / "build.log"
    log.write_text(" ".join(cmd) + "\n\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr)
        raise RuntimeError(f"nvcc failed (exit {res.returncode}); see {log}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
