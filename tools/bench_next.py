"""Measure the §8f consumers on one GPU (c2 text: n = 2^30 bytes, sigma = 256).

    python tools/bench_next.py [--steps 10] [--queries 16777216] > profiles/r1_next_bench.json

Prints one JSON object: per component the CUDA-event time per call (median of
`--steps` after 3 warm-ups, inputs resident in HBM), its algorithmic bytes and
the fraction of the measured HBM peak, and batched query throughput.
  directory : wvlt_rank_select_build over the 8 matrix levels (reads the level
              words, writes superblock / block / sample arrays)
  convert   : WT -> WM level reordering (levels 2..7 through wvlt_merge_bits,
              levels 0-1 copied): reads + writes every level once
  queries   : wvlt_query access / rank / select, random positions / symbols
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402
from paper_1702_07578_b200.support import DeviceDirectory, DeviceSupport, directory_shape  # noqa: E402
from paper_1702_07578_b200.wt2wm import ConversionPlan, convert_levels_device  # noqa: E402


def peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 7700.0, "fallback (B200_PROFILING.md HBM3e nominal)"


def timed(fn, steps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--queries", type=int, default=1 << 24)
    a = ap.parse_args()
    cfg = workloads.CONFIGS["c2"]
    n, sigma = cfg["n"], cfg["sigma"]
    text = workloads.generate("c2")
    b = DeviceBuilder()
    peak, src = peak_gbs()
    res = {"workload": "c2 (WM/WT, n=2^30 u8, sigma=256, Zipf 1.1); synthetic, inputs resident in HBM",
           "peak_gbs": peak, "peak_source": src}

    wm = b.build(text, sigma, "wm")
    width = wm.width
    nwords, nsuper, nblocks, nsamp = directory_shape(n)
    ms = timed(lambda: DeviceDirectory(wm.level_words, width, n), a.steps)
    byts = width * (nwords * 8 + nsuper * 8 + nblocks * 8) + width * nsamp * 16
    res["directory"] = {"ms": ms, "algorithmic_bytes": byts, "gbs": byts / ms / 1e6,
                        "frac": byts / ms / 1e6 / peak, "levels": width}

    wt = b.build(text, sigma, "wt", histogram=True)
    hist = wt.hist.cpu().numpy()
    ms = timed(lambda: convert_levels_device(wt.level_words, n, sigma, hist, builder=b), a.steps)
    byts = 2 * width * nwords * 8
    res["convert"] = {"ms": ms, "algorithmic_bytes": byts, "gbs": byts / ms / 1e6,
                      "frac": byts / ms / 1e6 / peak, "includes": "plan build + one H2D of all level plans"}
    plan = ConversionPlan(hist, n, sigma, wt.level_words.device)
    out = torch.empty_like(wt.level_words)
    ms = timed(lambda: plan.run(wt.level_words, out, b), a.steps)
    res["convert_kernels"] = {"ms": ms, "gbs": byts / ms / 1e6, "frac": byts / ms / 1e6 / peak,
                              "includes": "2 level copies + 6 wvlt_merge_bits launches, plan resident"}
    del wt

    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    q = a.queries
    pos = torch.randint(0, n, (q,), generator=g, device="cuda", dtype=torch.int64)
    for kind in ("wm", "wt"):
        st = wm if kind == "wm" else b.build(text, sigma, "wt")
        ds = DeviceSupport.from_build(st)
        syms = text[pos[: q]].to(torch.int64)
        r = ds.rank(syms, pos)
        entry = {}
        entry["access"] = q / (timed(lambda: ds.access(pos), a.steps) * 1e-3)
        entry["rank"] = q / (timed(lambda: ds.rank(syms, pos), a.steps) * 1e-3)
        entry["select"] = q / (timed(lambda: ds.select(syms, r + 1), a.steps) * 1e-3)
        assert torch.equal(ds.access(pos[:4096]), syms[:4096])
        res[f"queries_{kind}_per_s"] = entry
    res["queries"] = q
    print(json.dumps(res))


if __name__ == "__main__":
    main()
