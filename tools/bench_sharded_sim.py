"""Device-side cost of the sharded (multi-GPU) build, measured on ONE GPU.

    python tools/bench_sharded_sim.py [--configs c2 c4 c5] [--ranks 2 4 8] [--log2n N]

Only one GPU is available to this project, so the N-GPU bench path (bench.py --gpus N
under torchrun) cannot be timed.  What CAN be timed on one GPU is every device
kernel a rank runs in the p2p transport (distributed._build_sharded_p2p), one rank
after another, with all "peer" buffers in the same HBM:

  local   the rank's build of its shard (levels + histogram + node borders + zeros)
  plan    wvlt_peer_plan: every level's merge plan from the stacked
          [histogram | borders | zeros | flag] rows (what the all_gather returns)
  merge   wvlt_merge_levels_peer: the owner assembles its word range of every level
          from the R local level sets

The ranks run sequentially (no kernel waits on another rank), and the owners'
word ranges are checked against the single build.  This is NOT an NVLink
measurement: peer reads are HBM-local here, and the two small collectives
(all_gather of the rows, the completion all_reduce) are not included.  The line
gives the per-rank device time an R-GPU run would spend outside NVLink
(max local + plan + max merge) and the merge kernel's bandwidth against the
HBM peak.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1702_07578_b200.bitperm import code_width  # noqa: E402
from paper_1702_07578_b200.distributed import CudaOps, word_ranges  # noqa: E402


def timed(fn, reps=3):
    """median CUDA-event time of fn() in ms (one warm-up)"""
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def peak_gbs():
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def run(config: str, world: int, n: int | None, verify: bool):
    cfg = workloads.CONFIGS[config]
    n = n or cfg["n"]
    sigma, kind = cfg["sigma"], cfg["kind"]
    width = code_width(sigma)
    nb = 1 << width
    nbd = max(nb - 2, 0)
    text = workloads.generate(config, n=n)
    dev = text.device
    ops = CudaOps()
    # position shards: multiples of 512 symbols like construct._aligned_slices (construct.py:199-211)
    chunk = -(-(-(-n // world)) // 512) * 512
    cuts = [min(r * chunk, n) for r in range(world + 1)]
    lns = [cuts[r + 1] - cuts[r] for r in range(world)]
    lnws = [(v + 63) >> 6 for v in lns]
    total_words = (n + 63) >> 6
    ranges = word_ranges(total_words, world)
    # every rank's "peer-visible" level buffer (one allocation each, as the symmetric-memory buffers are)
    bufs = [torch.empty(width * max(lnws), dtype=torch.int64, device=dev) for _ in range(world)]
    rows = [None] * world
    t_local = []
    for r in range(world):
        shard = text[cuts[r]:cuts[r + 1]]

        def local():
            lw, hist, bad, borders, zeros_local = ops.local_build(shard, sigma, kind,
                                                                  out_words=bufs[r][: width * lnws[r]], borders=True)
            flag = (bad.reshape(-1)[:1].to(torch.int64) & 1)
            rows[r] = torch.cat([hist.reshape(-1).to(torch.int64), borders.reshape(-1)[:nbd].to(torch.int64),
                                 zeros_local.reshape(-1)[:width].to(torch.int64), flag.reshape(-1)])

        t_local.append(timed(local))
    allrows = torch.stack(rows).contiguous()
    rowlen = allrows.shape[1]
    ns = torch.tensor(lns, dtype=torch.int64, device=dev)
    plan = None

    def do_plan():
        nonlocal plan
        plan = ops.device_plan(allrows, rowlen, nb, ns, world, width, kind)

    t_plan = timed(do_plan)
    level_src = ops.level_sources([int(b.data_ptr()) for b in bufs], lnws, width, world)
    owned = [torch.empty((width, max(w1 - w0, 0)), dtype=torch.int64, device=dev) for (w0, w1) in ranges]
    t_merge = []
    for o, (w0, w1) in enumerate(ranges):
        t_merge.append(timed(lambda: ops.merge_peer_device(owned[o], w0, w1, n, plan, level_src, world)))
    ok = None
    if verify:
        del bufs
        want = ops.builder.build(text, sigma, kind).level_words
        ok = all(torch.equal(owned[o], want[:, w0:w1]) for o, (w0, w1) in enumerate(ranges))
        del want
    single = timed(lambda: ops.builder.build(text, sigma, kind, check=False))
    # merge traffic per owner: its destination words written once + the same number of source bits read
    merge_bytes = 2 * 8 * width * max(w1 - w0 for (w0, w1) in ranges)
    worst = max(t_merge)
    per_rank = max(t_local) + t_plan + worst
    out = {
        "config": config, "kind": kind, "n": n, "sigma": sigma, "levels": width, "ranks": world,
        "local_build_ms": {"max": round(max(t_local), 4), "mean": round(sum(t_local) / world, 4)},
        "plan_ms": round(t_plan, 4),
        "merge_ms": {"max": round(worst, 4), "mean": round(sum(t_merge) / world, 4)},
        "merge_gbs": round(merge_bytes / worst / 1e6, 1),
        "merge_frac_of_hbm_peak": round(merge_bytes / worst / 1e6 / peak_gbs(), 3),
        "per_rank_device_ms": round(per_rank, 4),
        "single_gpu_build_ms": round(single, 4),
        "device_speedup_vs_single": round(single / per_rank, 2),
        "verified_equal_to_single_build": ok,
        "note": "one GPU, ranks run one after another, peer reads are HBM-local: NOT an NVLink measurement; "
                "the rows all_gather and the completion all_reduce are not included",
    }
    print(json.dumps(out), flush=True)
    del owned, text
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["c2", "c4", "c5"])
    ap.add_argument("--ranks", nargs="*", type=int, default=[2, 4, 8])
    ap.add_argument("--log2n", type=int, default=None)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--variant", default=None, help="a tools/variants/<name>.so tuning build instead of the product library")
    a = ap.parse_args()
    if a.variant:
        from paper_1702_07578_b200 import _lib

        _lib.load_variant(ROOT / "tools" / "variants" / f"{a.variant}.so")
    for c in a.configs:
        for r in a.ranks:
            run(c, r, (1 << a.log2n) if a.log2n else None, not a.no_verify)


if __name__ == "__main__":
    main()
