"""Golden vectors for the consumers of a built structure, from the reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_next.py

Writes tests/golden/golden_next.npz.  Every expected value was produced by the
reference package ``wvlt`` itself:

* rank/select directories and answers: ``RankSelectBitVector`` (bitvec.py:118-263)
  on bit vectors shaped like test_bitvec.py's cases plus larger random ones;
* structure queries: ``access`` / ``rank`` / ``select`` of the tree and the
  matrix built by ``build_structure`` (structures.py:107-256), absent select
  occurrences recorded as -1;
* conversion: ``convert_wt_to_wm`` dumps, ``recover_histogram``,
  ``interval_start_table``, ``unary_histogram`` and ``TreeToMatrixMap``
  answers (wt2wm.py).

Inputs are seeded synthetic bit vectors and texts (no corpus data).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import wvlt  # noqa: E402
from wvlt.bitvec import AbsentOccurrenceError, BitVector, RankSelectBitVector  # noqa: E402
from wvlt.levelstats import symbol_histogram  # noqa: E402
from wvlt.wt2wm import (TreeToMatrixMap, convert_wt_to_wm, interval_start_table, recover_histogram,  # noqa: E402
                        unary_histogram)

OUT = Path(__file__).resolve().parent / "golden_next.npz"
SEED = 0x574C55


def bitvectors(rng):
    yield rng.integers(0, 2, 0, dtype=np.uint8)
    yield np.zeros(645, dtype=np.uint8)
    yield np.ones(645, dtype=np.uint8)
    yield rng.integers(0, 2, 63, dtype=np.uint8)
    yield rng.integers(0, 2, 64, dtype=np.uint8)
    yield rng.integers(0, 2, 2048 + 17, dtype=np.uint8)
    yield (rng.random(3 * 8192 + 77) < 0.9).astype(np.uint8)
    yield (rng.random(5000) < 0.01).astype(np.uint8)
    yield rng.integers(0, 2, 40_000, dtype=np.uint8)
    yield (rng.random(70_001) < 0.3).astype(np.uint8)


def main():
    rng = np.random.default_rng(SEED)
    out = {}
    # --- rank/select directories and answers
    for k, bits in enumerate(bitvectors(rng)):
        bv = BitVector.from_bits(bits)
        sup = RankSelectBitVector(bv)
        n = bits.size
        out[f"rs{k}_length"] = np.array([n], dtype=np.int64)
        out[f"rs{k}_words"] = bv.words.copy()
        out[f"rs{k}_super_zeros"] = np.asarray(sup._super_zeros, dtype=np.int64)
        out[f"rs{k}_block_zeros"] = np.asarray(sup._block_zeros, dtype=np.int64)
        out[f"rs{k}_samples1"] = np.asarray(sup._samples1, dtype=np.int64)
        out[f"rs{k}_samples0"] = np.asarray(sup._samples0, dtype=np.int64)
        out[f"rs{k}_ones"] = np.array([sup.count(1)], dtype=np.int64)
        probe = np.unique(np.concatenate((np.arange(0, n + 1, 97), [0, n], rng.integers(0, n + 1, 60))))
        out[f"rs{k}_rank_pos"] = probe.astype(np.int64)
        out[f"rs{k}_rank1"] = np.array([sup.rank(1, int(i)) for i in probe], dtype=np.int64)
        for x in (0, 1):
            total = sup.count(x)
            js = np.unique(np.concatenate((np.arange(1, total + 1, max(total // 60, 1)), [total, total + 1])))
            js = js[js >= 1]
            ans = []
            for j in js:
                try:
                    ans.append(sup.select(x, int(j)))
                except AbsentOccurrenceError:
                    ans.append(-1)
            out[f"rs{k}_sel{x}_j"] = js.astype(np.int64)
            out[f"rs{k}_sel{x}"] = np.array(ans, dtype=np.int64)
    out["rs_count"] = np.array([k + 1], dtype=np.int64)

    # --- structure queries and conversion
    cases = []
    for sigma in (1, 2, 5, 16, 200, 1000, 70000):
        for n in (0, 1, 777, 3000):
            cases.append((sigma, n))
    for ci, (sigma, n) in enumerate(cases):
        dt = np.uint8 if sigma <= 256 else np.uint16 if sigma <= 65536 else np.uint32
        text = rng.integers(0, sigma, n).astype(dt) if sigma > 1 else np.zeros(n, dtype=dt)
        if sigma >= 16 and n:  # skew: a few heavy symbols and absent ones
            text[rng.random(n) < 0.4] = dt(sigma // 3)
        out[f"q{ci}_sigma"] = np.array([sigma], dtype=np.int64)
        out[f"q{ci}_text"] = text
        pos = rng.integers(0, max(n, 1), 50).astype(np.int64) if n else np.zeros(0, dtype=np.int64)
        rpos = rng.integers(0, n + 1, 50).astype(np.int64)
        syms = rng.integers(0, sigma, 50).astype(np.int64)
        syms[:5] = sigma // 3
        js = rng.integers(1, max(n // 4, 2) + 1, 50).astype(np.int64)
        out[f"q{ci}_pos"] = pos
        out[f"q{ci}_rpos"] = rpos
        out[f"q{ci}_syms"] = syms
        out[f"q{ci}_js"] = js
        for kind in ("wt", "wm"):
            st = wvlt.build_structure(text, sigma, kind)
            out[f"q{ci}_{kind}_access"] = np.array([st.access(int(i)) for i in pos], dtype=np.int64)
            out[f"q{ci}_{kind}_rank"] = np.array([st.rank(int(c), int(i)) for c, i in zip(syms, rpos)],
                                                 dtype=np.int64)
            sel = []
            for c, j in zip(syms, js):
                try:
                    sel.append(st.select(int(c), int(j)))
                except AbsentOccurrenceError:
                    sel.append(-1)
            out[f"q{ci}_{kind}_select"] = np.array(sel, dtype=np.int64)
        wt = wvlt.build_structure(text, sigma, "wt")
        wm = convert_wt_to_wm(wt)
        out[f"q{ci}_conv_dump"] = np.frombuffer(wvlt.dump_structure(wm), dtype=np.uint8).copy()
        out[f"q{ci}_recovered"] = np.asarray(recover_histogram(wt), dtype=np.int64)
        hist = symbol_histogram(text, sigma) if n else np.zeros(1 << wvlt.code_width(sigma), dtype=np.int64)
        out[f"q{ci}_start_table"] = np.asarray(interval_start_table(hist, sigma), dtype=np.int64)
        if n:
            m = TreeToMatrixMap(hist, sigma)
            lv = rng.integers(0, max(m.width, 1), 40) if m.width else np.zeros(0, dtype=np.int64)
            ip = rng.integers(0, n, lv.size)
            out[f"q{ci}_map_level"] = lv.astype(np.int64)
            out[f"q{ci}_map_pos"] = ip.astype(np.int64)
            out[f"q{ci}_map"] = np.array([m.map_position(int(a), int(b)) for a, b in zip(lv, ip)], dtype=np.int64)
        uh = unary_histogram(hist[:sigma] if sigma <= hist.size else hist)
        out[f"q{ci}_unary_len"] = np.array([uh.length], dtype=np.int64)
        out[f"q{ci}_unary_words"] = uh.words.copy()
    out["q_count"] = np.array([len(cases)], dtype=np.int64)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
