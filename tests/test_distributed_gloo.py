"""Sharded multi-GPU build: host plan + collectives, on CPU with gloo.

The product path (distributed.build_sharded) runs the local builds and the
shift-merge on the GPU and the collectives over NCCL.  Here every rank is a
CPU process on the gloo backend; the oracle (test infrastructure) stands in
for the two device kernels so the exchange plan, the all_gather of
histograms, the all_to_all of bit segments and the merge bookkeeping are
exercised for real.  The assembled structure must equal the single build.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleOps:
    """CPU stand-ins for the local device build and wvlt_merge_bits."""

    def __init__(self):
        import torch

        self.device = torch.device("cpu")

    def local_build(self, text, sigma, kind):
        import torch

        import oracle

        arr = np.asarray(text)
        words, _, hist = oracle.build(arr, sigma, kind, "pc")
        if hist is None or arr.size == 0:
            hist = oracle.histogram(arr, sigma)
        return (torch.from_numpy(np.ascontiguousarray(words).view(np.int64)),
                torch.from_numpy(np.ascontiguousarray(hist, dtype=np.int64)), False)

    def merge(self, dst_row, word_lo, word_hi, n_bits, bounds, src_starts, src):
        import torch

        import oracle

        full = oracle.merge_bits(n_bits, bounds, src_starts, src.numpy().view(np.uint64), word_lo, word_hi)
        dst_row.copy_(torch.from_numpy(full[word_lo:word_hi].view(np.int64)))


def _worker(rank, world, port, cases, out_dir):
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1702_07578_b200.distributed import build_sharded

    import oracle

    results = []
    for ci, (n, sigma, kind, cuts) in enumerate(cases):
        rng = np.random.default_rng(1000 + ci)
        text = rng.integers(0, sigma, n).astype(np.uint32 if sigma > 65536 else np.uint16 if sigma > 256 else np.uint8)
        lo, hi = cuts[rank], cuts[rank + 1]
        res = build_sharded(text[lo:hi], sigma, kind, ops=OracleOps(), gather=True)
        if rank == 0:
            words, zeros, _ = oracle.build(text, sigma, kind, "pc")
            got = res.full_words.numpy().view(np.uint64)
            ok = np.array_equal(got, words) and (kind == "wt" or list(res.zeros) == list(zeros))
            results.append((ci, bool(ok)))
    if rank == 0:
        np.save(os.path.join(out_dir, "results.npy"), np.array(results, dtype=np.int64))
    dist.destroy_process_group()


def _cases(world, rng):
    cases = []
    for sigma in (2, 5, 256, 1000, 70000):
        for kind in ("wt", "wm"):
            n = int(rng.integers(3000, 20000))
            inner = sorted(int(v) for v in rng.integers(0, n, world - 1))
            if sigma == 5:  # an empty shard and a shard boundary inside a word
                inner = [0] + inner[1:] if world > 2 else [129]
            cases.append((n, sigma, kind, [0] + inner + [n]))
    return cases


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_build_matches_single_build(world, tmp_path):
    import torch.multiprocessing as mp

    cases = _cases(world, np.random.default_rng(world))
    mp.start_processes(_worker, args=(world, _free_port(), cases, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = np.load(tmp_path / "results.npy")
    assert len(res) == len(cases)
    bad = [int(ci) for ci, ok in res if not ok]
    assert not bad, [cases[i][:3] for i in bad]


def test_level_plan_matches_reference_merge_order():
    """Plan pieces walk prefix groups in interval order, ranks in text order
    (construct._merge_plan, construct.py:516-543)."""
    from paper_1702_07578_b200.distributed import level_plan

    h = np.array([[1, 2, 0, 3, 1, 1, 0, 2], [0, 1, 4, 0, 2, 0, 1, 1]], dtype=np.int64)  # w = 3
    ranks, local, lens, gstart = level_plan(h, "wm", 3, 2)
    # 2-bit prefix counts per rank: r0 [3,3,2,2], r1 [1,4,2,2]; WM order rho_2 = [0,2,1,3]
    assert list(lens) == [3, 1, 2, 2, 3, 4, 2, 2]
    assert list(ranks) == [0, 1, 0, 1, 0, 1, 0, 1]
    assert list(local) == [0, 0, 3, 1, 5, 3, 8, 7]
    assert list(gstart) == [0, 3, 4, 6, 8, 11, 15, 17]
    ranks, local, lens, gstart = level_plan(h, "wt", 3, 2)
    assert list(lens) == [3, 1, 3, 4, 2, 2, 2, 2]


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("sigma,world", [(5, 2), (256, 3), (1000, 4), (70000, 3)])
def test_peer_merge_plan_reassembles_the_single_build(kind, sigma, world):
    """The p2p transport's per-owner task arrays (peer_plan_arrays), applied by the
    host restatement of wvlt_merge_levels_peer to every rank's local levels,
    reassemble the single build (no process group needed: the plan is pure)."""
    import oracle
    from paper_1702_07578_b200.bitperm import code_width
    from paper_1702_07578_b200.distributed import exchange_plan, merge_peer_host, peer_plan_arrays

    rng = np.random.default_rng(sigma + world)
    n = 3000 + 7 * world
    text = rng.integers(0, sigma, n).astype(np.uint32 if sigma > 65536 else np.uint16 if sigma > 256 else np.uint8)
    cuts = [0] + sorted(rng.choice(np.arange(1, n), world - 1, replace=False).tolist()) + [n]
    width = code_width(sigma)
    sources, hists = [], []
    for r in range(world):
        part = text[cuts[r]:cuts[r + 1]]
        w, _, h = oracle.build(part, sigma, kind, "pc")
        sources.append(np.asarray(w, dtype=np.uint64))
        hists.append(oracle.histogram(part, sigma) if h is None else np.asarray(h, dtype=np.int64))
    ranges, plans = exchange_plan(np.stack(hists), kind, width, n, [cuts[r + 1] - cuts[r] for r in range(world)],
                                  world)
    want, _, _ = oracle.build(text, sigma, kind, "pc")
    for owner, (w0, w1) in enumerate(ranges):
        arrays = peer_plan_arrays(plans, owner, width)
        got = merge_peer_host(arrays, sources, w0, w1, n, width)
        assert np.array_equal(got, np.asarray(want, dtype=np.uint64)[:, w0:w1]), owner


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("width", [1, 3, 8])
def test_owner_plan_equals_full_exchange_plan(kind, world, width):
    """owner_plan_arrays (the p2p path computes only its own merge tasks) equals
    the owner's slice of the full exchange plan, skewed and empty groups included."""
    from paper_1702_07578_b200.distributed import exchange_plan, owner_plan_arrays, peer_plan_arrays

    rng = np.random.default_rng(world * 100 + width)
    hists = (rng.zipf(1.3, (world, 1 << width)) % 5000).astype(np.int64)
    hists[:, rng.integers(0, 1 << width, max(1, (1 << width) // 4))] = 0
    local_ns = [int(h.sum()) for h in hists]
    n = sum(local_ns)
    _, plans = exchange_plan(hists, kind, width, n, local_ns, world)
    for owner in range(world):
        want = peer_plan_arrays(plans, owner, width)
        got = owner_plan_arrays(hists, kind, width, n, owner, world)
        for a, b in zip(want, got):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("width", [1, 2, 3, 8, 12])
def test_device_plan_restatement_equals_merge_plan(kind, world, width):
    """The device plan (wvlt_peer_plan, restated by plan_from_borders_host) built from
    the ranks' node borders has, per level, exactly the pieces of the reference
    merge plan (construct._merge_plan, construct.py:516-543 -> level_plan) once
    the empty ones are dropped; the merge it drives (host restatement of
    merge_peer_kernel) gives the single build's words for every owner."""
    import oracle
    from paper_1702_07578_b200.distributed import level_plan, merge_peer_host, plan_from_borders_host, word_ranges

    rng = np.random.default_rng(world * 1000 + width * 7 + (kind == "wm"))
    sigma = 1 << width
    n = int(rng.integers(2000, 6000))
    text = (rng.zipf(1.3, n) % sigma).astype(np.uint16 if width > 8 else np.uint8)
    cuts = [0] + sorted(int(v) for v in rng.integers(0, n, world - 1)) + [n]
    if world > 2:
        cuts[1] = 0  # an empty shard
    shards = [text[cuts[r]:cuts[r + 1]] for r in range(world)]
    hists = np.stack([oracle.histogram(s, sigma) for s in shards])
    borders = [oracle.borders(h, width, kind) for h in hists]
    local_ns = [s.size for s in shards]
    bounds, boff, starts, ranks, toff = plan_from_borders_host(borders, local_ns, kind, width)
    for ell in range(width):
        t0, t1 = int(toff[ell]), int(toff[ell + 1])
        b = bounds[int(boff[ell]): int(boff[ell]) + (t1 - t0) + 1]
        lens = np.diff(b)
        keep = lens > 0
        pr, pl, pn, pg = level_plan(hists, kind, width, ell)
        assert np.array_equal(ranks[t0:t1][keep], pr)
        assert np.array_equal(starts[t0:t1][keep], pl)
        assert np.array_equal(lens[keep], pn)
        assert np.array_equal(b[:-1][keep], pg)
        assert int(b[-1]) == n
    sources = [oracle.build(s, sigma, kind, "pc")[0] for s in shards]
    want, _, _ = oracle.build(text, sigma, kind, "pc")
    for owner, (w0, w1) in enumerate(word_ranges((n + 63) >> 6, world)):
        got = merge_peer_host((bounds, boff, starts, ranks, toff), sources, w0, w1, n, width)
        assert np.array_equal(got, np.asarray(want, dtype=np.uint64)[:, w0:w1]), owner
