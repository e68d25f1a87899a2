"""Generate golden vectors for the construction path by running the reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Every expected value in it was produced by
the reference package ``wvlt`` itself:

* ``dump_structure(build_by_prefix_counting(text, sigma, kind))``
  (construct.py:292-319, structures.py:259-278), cross-checked against the
  reference's brute-force ``naive_structure`` (oracle.py:87-97) where that
  accepts the input and against ``ps`` at 3 threads;
* ``symbol_histogram`` (levelstats.py:30-47);
* node borders per level: ``interval_starts`` of the folded histogram
  (levelstats.py:58-73) for the tree and ``interval_start_table``
  (wt2wm.py:55-78) for the matrix;
* ``gather_bits`` (_kernels.py:196-232) on random interval plans.

Inputs are seeded synthetic texts (no corpus data).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import wvlt  # noqa: E402
from wvlt import _kernels  # noqa: E402
from wvlt.levelstats import fold_histogram, interval_starts, symbol_histogram  # noqa: E402
from wvlt.oracle import MAX_ORACLE_N, MAX_ORACLE_SIGMA, naive_structure  # noqa: E402
from wvlt.wt2wm import interval_start_table  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"
SEED = 0x574C54


def dtype_for(sigma: int):
    if sigma <= 1 << 8:
        return np.uint8
    if sigma <= 1 << 16:
        return np.uint16
    return np.uint32


def make_text(rng, n: int, sigma: int, dist: str) -> np.ndarray:
    dt = dtype_for(sigma)
    if sigma <= 1 or n == 0:
        return np.zeros(n, dtype=dt)
    if dist == "uniform":
        return rng.integers(0, sigma, n, dtype=dt)
    if dist == "zipf":
        ranks = np.arange(1, sigma + 1, dtype=np.float64)
        p = ranks ** -1.1
        p /= p.sum()
        perm = rng.permutation(sigma)
        return perm[rng.choice(sigma, n, p=p)].astype(dt)
    if dist == "const":
        return np.full(n, sigma - 1, dtype=dt)
    if dist == "sorted":
        return np.sort(rng.integers(0, sigma, n, dtype=dt))
    if dist == "runs":  # long runs of one symbol: tiles spanning one / many nodes
        out = np.empty(n, dtype=dt)
        i = 0
        while i < n:
            ln = int(rng.integers(1, 3000))
            out[i : i + ln] = rng.integers(0, sigma)
            i += ln
        return out
    if dist == "sparse":  # few distinct symbols spread over a wide alphabet
        vals = rng.choice(sigma, size=min(sigma, 7), replace=False)
        return vals[rng.integers(0, vals.size, n)].astype(dt)
    raise ValueError(dist)


def borders_of(hist, sigma: int, kind: str) -> np.ndarray:
    w = wvlt.code_width(sigma)
    if kind == "wm":
        return interval_start_table(hist, sigma)
    out = np.zeros(max((1 << w) - 2, 0), dtype=np.int64)
    h = np.asarray(hist, dtype=np.int64)
    for ell in range(w - 1, 0, -1):
        h = fold_histogram(h)
        out[(1 << ell) - 2 : (1 << (ell + 1)) - 2] = interval_starts(h)
    return out


def cases():
    rng = np.random.default_rng(SEED)
    tile_ns = [0, 1, 2, 31, 32, 33, 63, 64, 65, 511, 512, 513, 4095, 4096, 4097, 8191, 8192, 8193, 12289, 16385]
    out = []
    # every sigma of the reference SIGMA_GRID (conftest.py:6) plus the configs' alphabets
    for sigma in (1, 2, 3, 4, 5, 16, 200, 256, 1000, 65536, 70000, 1 << 20):
        ns = tile_ns if sigma in (5, 256, 70000) else [0, 1, 65, 4097, 8193, int(rng.integers(100, 20000))]
        for i, n in enumerate(ns):
            dist = ("uniform", "zipf", "runs", "sparse", "sorted", "const")[i % 6]
            out.append((n, sigma, dist))
    # larger cases crossing many tiles
    for sigma, dist in ((256, "zipf"), (256, "runs"), (5, "uniform"), (4, "runs"), (65536, "zipf"),
                        (1 << 20, "uniform"), (1000, "sparse")):
        out.append((int(rng.integers(40_000, 70_000)) if sigma <= 1000 else int(rng.integers(20_000, 30_000)),
                    sigma, dist))
    return rng, out


def main():
    rng, spec = cases()
    arrays = {}
    meta = []
    for ci, (n, sigma, dist) in enumerate(spec):
        text = make_text(rng, n, sigma, dist)
        arrays[f"text_{ci}"] = text
        hist = symbol_histogram(text, sigma)
        arrays[f"hist_{ci}"] = hist
        for kind in ("wt", "wm"):
            st = wvlt.build_by_prefix_counting(text, sigma, kind)
            blob = wvlt.dump_structure(st)
            if n <= 20_000 and sigma <= MAX_ORACLE_SIGMA and n <= MAX_ORACLE_N:
                assert wvlt.dump_structure(naive_structure(text, sigma, kind)) == blob, (ci, kind)
            assert wvlt.dump_structure(wvlt.build_structure(text, sigma, kind, "ps", 3)) == blob, (ci, kind)
            arrays[f"dump_{kind}_{ci}"] = np.frombuffer(blob, dtype=np.uint8)
            if wvlt.code_width(sigma) <= 12:  # keep the fixture small; wide alphabets are pinned by dumps
                arrays[f"borders_{kind}_{ci}"] = borders_of(hist, sigma, kind)
        meta.append((n, sigma, dist))
    arrays["case_n"] = np.array([m[0] for m in meta], dtype=np.int64)
    arrays["case_sigma"] = np.array([m[1] for m in meta], dtype=np.int64)
    arrays["case_dist"] = np.array([m[2] for m in meta])

    # running example, SPEC/reference tests (test_acceptance.py:85-100)
    ex = np.array([0, 1, 6, 7, 1, 5, 4, 2, 6, 3], dtype=np.uint8)
    arrays["example_text"] = ex
    for kind in ("wt", "wm"):
        st = wvlt.build_by_prefix_counting(ex, 8, kind)
        arrays[f"example_words_{kind}"] = np.array([int(v.words[0]) for v in st.levels], dtype=np.uint64)
        arrays[f"example_dump_{kind}"] = np.frombuffer(wvlt.dump_structure(st), dtype=np.uint8)
    arrays["example_zeros"] = np.array(wvlt.build_by_prefix_counting(ex, 8, "wm").zeros, dtype=np.int64)

    # gather_bits on random plans (the multi-GPU merge / wt2wm kernel)
    for gi in range(6):
        n_bits = int(rng.integers(1, 5000))
        nsrc = int(rng.integers(n_bits, n_bits + 500))
        src = rng.integers(0, 2**63, (nsrc + 63) >> 6, dtype=np.uint64) | rng.integers(0, 2, (nsrc + 63) >> 6, dtype=np.uint64)
        cuts = np.unique(np.concatenate(([0, n_bits], rng.integers(1, n_bits, int(rng.integers(0, 60)))))) if n_bits > 1 else np.array([0, n_bits])
        lens = np.diff(cuts)
        starts = np.array([int(rng.integers(0, nsrc - ln + 1)) for ln in lens], dtype=np.int64)
        dst = np.zeros((n_bits + 63) >> 6, dtype=np.uint64)
        _kernels.gather_bits(dst, 0, dst.size, n_bits, cuts.astype(np.int64), starts, src, 0)
        arrays[f"gather_{gi}_nbits"] = np.array([n_bits], dtype=np.int64)
        arrays[f"gather_{gi}_bounds"] = cuts.astype(np.int64)
        arrays[f"gather_{gi}_starts"] = starts
        arrays[f"gather_{gi}_src"] = src
        arrays[f"gather_{gi}_dst"] = dst

    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(meta)} cases)")


if __name__ == "__main__":
    main()
