"""Parity of the CUDA path against the oracle and the reference's golden vectors.

Every build here goes through the product API / C ABI on the GPU; the oracle
(oracle/) and tests/golden (produced by the reference) are the checkers.
Integer path: bit-exact equality of the wire-format bytes is required.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_1702_07578_b200 as wv
from conftest import EXAMPLE_SIGMA, EXAMPLE_TEXT, SIGMA_GRID, dtype_for, golden, golden_cases, random_text

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

CASES = golden_cases()


def ref_dump(text, sigma, kind):
    words, zeros, _ = oracle.build(text, sigma, kind, "pc")
    return oracle.dump(kind, int(np.asarray(text).size), max(int(sigma), 1), words, zeros)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_golden_cases_bit_exact(kind):
    g = golden()
    for ci, n, sigma, dist in CASES:
        st = wv.build_structure(g[f"text_{ci}"], sigma, kind)
        assert wv.dump_structure(st) == g[f"dump_{kind}_{ci}"].tobytes(), (ci, n, sigma, dist)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_golden_node_borders_from_drop_in(kind):
    """build_structure(...).node_borders(l) == the reference's interval_starts of the
    folded histogram (WT, levelstats.py:58-73) / interval_start_table block l (WM,
    wt2wm.py:55-78), for every golden case and level (code widths above 12 carry
    no golden borders: the oracle's restatement, pinned to the golden ones, of the
    reference's golden histogram stands in)."""
    g = golden()
    for ci, n, sigma, dist in CASES:
        st = wv.build_structure(g[f"text_{ci}"], sigma, kind)
        key = f"borders_{kind}_{ci}"
        want = g[key] if key in g else oracle.borders(g[f"hist_{ci}"], wv.code_width(sigma), kind)
        w = wv.code_width(sigma)
        assert st.borders is not None and st.borders.shape == want.shape, (ci, n, sigma)
        for ell in range(1, w):
            assert np.array_equal(st.node_borders(ell), want[(1 << ell) - 2 : (1 << (ell + 1)) - 2]), (ci, ell)
        with pytest.raises(IndexError):
            st.node_borders(0)


@pytest.mark.parametrize("sigma", [4, 5, 256, 1000, 1 << 16, 70000, 1 << 20])
@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_node_borders_vs_oracle(kind, sigma):
    """Borders of larger texts through the drop-in (byte texts: the fused pass's
    tables; wider alphabets: the group recurrence over the matrix levels)."""
    rng = np.random.default_rng(sigma + 3)
    for n in (16385, 300_001):
        text = random_text(rng, n, sigma)
        st = wv.build_structure(text, sigma, kind)
        w = wv.code_width(sigma)
        assert np.array_equal(st.borders, oracle.borders(oracle.histogram(text, sigma), w, kind))
        assert wv.dump_structure(st) == ref_dump(text, sigma, kind)


def test_running_example():
    wt = wv.build_structure(EXAMPLE_TEXT, EXAMPLE_SIGMA, "wt")
    wm = wv.build_structure(EXAMPLE_TEXT, EXAMPLE_SIGMA, "wm")
    assert tuple(int(v.words[0]) for v in wt.levels) == (0x16C, 0x278, 0x136)
    assert tuple(int(v.words[0]) for v in wm.levels) == (0x16C, 0x278, 0x14E)
    assert wm.zeros == [5, 5, 5]


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("sigma", SIGMA_GRID + (4, 17, 33, 100, 256, 1000, 1 << 16, (1 << 17) + 5, 1 << 20, 1 << 24))
def test_tile_boundaries_vs_oracle(kind, sigma):
    rng = np.random.default_rng(sigma * 7 + (kind == "wm"))
    for n in (1, 31, 32, 33, 63, 64, 65, 4095, 4096, 4097, 8191, 8192, 8193, 16383, 16384, 16385, 32767, 32768, 32769, 40961, 49153,
              int(rng.integers(100_000, 300_000))):
        text = random_text(rng, n, sigma)
        assert wv.dump_structure(wv.build_structure(text, sigma, kind)) == ref_dump(text, sigma, kind), (n, sigma)


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_distributions_vs_oracle(kind):
    """Skewed / clustered inputs: Zipf heavy hitters, long runs (tiles inside one
    node and tiles spanning many nodes), sorted, few distinct symbols."""
    rng = np.random.default_rng(11)
    for sigma in (5, 256, 1000, 70000, 1 << 20):
        n = 200_003
        dt = dtype_for(sigma)
        ranks = rng.zipf(1.1, n) % sigma
        perm = rng.permutation(sigma)
        texts = {
            "zipf": perm[ranks].astype(dt),
            "runs": np.repeat(rng.integers(0, sigma, 200), rng.integers(1, 2000, 200))[:n].astype(dt),
            "sorted": np.sort(rng.integers(0, sigma, n)).astype(dt),
            "sparse": rng.choice(rng.choice(sigma, min(sigma, 3), replace=False), n).astype(dt),
            "const": np.full(n, sigma - 1, dtype=dt),
        }
        for name, text in texts.items():
            assert wv.dump_structure(wv.build_structure(text, sigma, kind)) == ref_dump(text, sigma, kind), (
                sigma, name)


def test_input_dtypes_and_layouts(rng):
    # test_construct.py:64-72: list, int32, uint64, strided, plus wider-than-needed storage
    base = random_text(rng, 5000, 16)
    ref = ref_dump(base, 16, "wt")
    assert wv.dump_structure(wv.build_by_prefix_counting(list(map(int, base)), 16, "wt")) == ref
    for dt in (np.int32, np.uint64, np.uint16, np.uint32, np.int64):
        assert wv.dump_structure(wv.build_by_prefix_counting(base.astype(dt), 16, "wt")) == ref, dt
    strided = np.repeat(base, 2)[::2]
    assert wv.dump_structure(wv.build_by_prefix_counting(strided, 16, "wt")) == ref
    # u8 storage with a wide alphabet
    small = random_text(rng, 9000, 256)
    assert wv.dump_structure(wv.build_structure(small, 70000, "wm")) == ref_dump(small, 70000, "wm")
    assert wv.dump_structure(wv.build_structure(small, 70000, "wt")) == ref_dump(small, 70000, "wt")


def test_every_algorithm_and_thread_count_is_identical(rng):
    # test_construct.py:43-51
    for sigma in (2, 16, 70000):
        text = random_text(rng, int(rng.integers(500, 30000)), sigma)
        for kind in ("wt", "wm"):
            ref = ref_dump(text, sigma, kind)
            for algo in wv.ALGORITHMS:
                for p in (1, 3, 8):
                    assert wv.dump_structure(wv.build_structure(text, sigma, kind, algo, p)) == ref


def test_out_of_range_symbols_raise(rng):
    for sigma, dt in ((5, np.uint8), (200, np.uint8), (1000, np.uint16), (70000, np.uint32), (256, np.uint16)):
        text = random_text(rng, 100_000, sigma).astype(dt)
        text[77_777] = sigma
        with pytest.raises(ValueError):
            wv.build_structure(text, sigma, "wm")
        with pytest.raises(ValueError):
            wv.build_structure(text, sigma, "wt")


def test_histogram_zeros_and_borders_vs_oracle(rng):
    from paper_1702_07578_b200.device import default_builder

    b = default_builder()
    for sigma in (3, 5, 256, 1000, 70000):
        text = random_text(rng, 300_000, sigma)
        t = torch.from_numpy(text).cuda()
        hist = oracle.histogram(text, sigma)
        w = wv.code_width(sigma)
        for kind in ("wt", "wm"):
            res = b.build(t, sigma, kind, borders=True, histogram=True)
            words, zeros, h = res.to_host()
            assert np.array_equal(h, hist)
            _, ozeros, _ = oracle.build(text, sigma, "wm", "pc")
            assert zeros == ozeros
            # histogram-free build (WM default): same words and zero counts
            lw, lz, lh = b.build(t, sigma, kind).to_host()
            assert lh is None
            assert np.array_equal(lw, words) and lz == zeros
            if w >= 2:
                assert np.array_equal(res.borders.cpu().numpy()[: (1 << w) - 2], oracle.borders(hist, w, kind))


def test_merge_bits_vs_reference_golden():
    from paper_1702_07578_b200.device import default_builder

    b = default_builder()
    g = golden()
    for gi in range(6):
        nbits = int(g[f"gather_{gi}_nbits"][0])
        nw = (nbits + 63) >> 6
        dst = torch.full((nw,), -1, dtype=torch.int64, device="cuda")
        src = torch.from_numpy(g[f"gather_{gi}_src"].view(np.int64)).cuda()
        b.merge_bits(dst, 0, nw, nbits, torch.from_numpy(g[f"gather_{gi}_bounds"]).cuda(),
                     torch.from_numpy(g[f"gather_{gi}_starts"]).cuda(), src)
        assert np.array_equal(dst.cpu().numpy().view(np.uint64), g[f"gather_{gi}_dst"]), gi


def test_device_builds_are_deterministic(rng):
    from paper_1702_07578_b200.device import default_builder

    b = default_builder()
    text = torch.from_numpy(random_text(rng, 3_000_000, 256)).cuda()
    for kind in ("wt", "wm"):
        a = b.build(text, 256, kind).level_words.clone()
        for _ in range(3):
            assert torch.equal(b.build(text, 256, kind).level_words, a)


@pytest.mark.slow
def test_config_c1_vs_oracle():
    """c1: n=2^20 uint8 sigma=256 uniform (BASELINE.json configs[0])."""
    rng = np.random.default_rng(0x574C54)
    text = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    for kind in ("wt", "wm"):
        assert wv.dump_structure(wv.build_structure(text, 256, kind)) == ref_dump(text, 256, kind)


def test_sharded_build_world1_nccl_matches_single_build(rng):
    """The multi-GPU path (CUDA local build + wvlt_merge_bits + NCCL collectives) at world size 1."""
    import os

    import torch.distributed as dist

    from paper_1702_07578_b200.distributed import build_sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29733")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        for sigma, kind in ((256, "wm"), (256, "wt"), (70000, "wm"), (5, "wt")):
            text = random_text(rng, 123_457, sigma)
            res = build_sharded(torch.from_numpy(text).cuda(), sigma, kind, gather=True)
            words, zeros, _ = oracle.build(text, sigma, kind, "pc")
            assert np.array_equal(res.full_words.cpu().numpy().view(np.uint64), words), (sigma, kind)
            if kind == "wm":
                assert list(res.zeros) == zeros
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sigma", [17, 100, 200, 256, 1000])
def test_unaligned_device_text(sigma):
    """A device text that does not start on a 16-byte boundary: the staging and
    counting kernels take their element-wise paths (single-pass byte kernels
    included), with identical output."""
    from paper_1702_07578_b200.device import DeviceBuilder

    rng = np.random.default_rng(sigma)
    n = 3 * 16384 + 777
    base = random_text(rng, n + 1, sigma)
    dev = torch.from_numpy(base).cuda()[1:]  # offset by one element
    assert dev.data_ptr() % 16 != 0
    b = DeviceBuilder()
    for kind in ("wt", "wm"):
        words, zeros, _ = b.build(dev, sigma, kind).to_host()
        ow, oz, _ = oracle.build(base[1:], sigma, kind, "pc")
        assert np.array_equal(words, ow), kind
        if kind == "wm":
            assert zeros == oz


@pytest.mark.parametrize("sigma", [300, 1000, 5000, 1 << 16])
def test_byte_storage_wide_alphabet_device_text(sigma):
    """A device text stored narrower than the code width (u8 storage, w > 8 or u16
    storage at w = 16): the build widens it and runs the fused 2-byte pass and
    the byte tail; output equals the oracle's."""
    from paper_1702_07578_b200.device import DeviceBuilder

    rng = np.random.default_rng(sigma + 5)
    n = 5 * 8192 + 4321
    hi = min(sigma, 256 if sigma <= 5000 else sigma)
    host = rng.integers(0, hi, n).astype(np.uint8 if hi <= 256 else np.uint16)
    dev = torch.from_numpy(host).cuda()
    b = DeviceBuilder()
    words, zeros, _ = b.build(dev, sigma, "wm").to_host()
    ow, oz, _ = oracle.build(host, sigma, "wm", "pc")
    assert np.array_equal(words, ow)
    assert zeros == oz


def test_concurrent_builds_on_two_streams():
    """One builder, two streams in flight at once: every stream gets its own
    workspace, so the builds do not interfere."""
    from paper_1702_07578_b200.device import DeviceBuilder

    b = DeviceBuilder()
    g = torch.Generator(device="cuda")
    g.manual_seed(21)
    texts = [torch.randint(0, 256, (3_000_001,), generator=g, device="cuda", dtype=torch.int64).to(torch.uint8),
             torch.randint(0, 1000, (2_000_003,), generator=g, device="cuda", dtype=torch.int64).to(torch.uint16)]
    sigmas = [256, 1000]
    want = [b.build(t, sg, "wm").level_words.clone() for t, sg in zip(texts, sigmas)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(3):
        got = []
        for t, sg, s in zip(texts, sigmas, streams):
            s.wait_stream(torch.cuda.current_stream())
            got.append(b.build(t, sg, "wm", stream=s, check=False))
        torch.cuda.synchronize()
        for r, w in zip(got, want):
            assert torch.equal(r.level_words, w)


@pytest.mark.parametrize("sigma,kind", [(256, "wt"), (5, "wm"), (1000, "wm"), (1 << 20, "wm")])
def test_captured_build_replays(sigma, kind):
    """DeviceBuilder.capture: one CUDA-graph replay per build of a refilled input
    buffer gives the same words as a plain build."""
    from paper_1702_07578_b200.device import DeviceBuilder

    b = DeviceBuilder()
    dt = torch.uint8 if sigma <= 256 else torch.uint16 if sigma <= 65536 else torch.uint32
    n = 1 << 20
    g = torch.Generator(device="cuda")
    g.manual_seed(sigma)
    buf = torch.randint(0, sigma, (n,), generator=g, device="cuda", dtype=torch.int64).to(dt)
    cap = b.capture(buf, sigma, kind)
    for _ in range(3):
        buf.copy_(torch.randint(0, sigma, (n,), generator=g, device="cuda", dtype=torch.int64).to(dt))
        res = cap.replay()
        torch.cuda.synchronize()
        want = b.build(buf.clone(), sigma, kind)
        assert torch.equal(res.level_words, want.level_words)
        if kind == "wm":
            assert torch.equal(res.zeros, want.zeros)
        cap.check()


@pytest.mark.parametrize("sigma,dt", [(5, torch.uint8), (200, torch.uint8), (1000, torch.uint16),
                                      (300, torch.uint16), ((1 << 20) - 3, torch.uint32), (1 << 23, torch.uint32),
                                      (70000, torch.uint32)])
@pytest.mark.parametrize("kind", ["wm", "wt"])
def test_device_range_check_every_path(sigma, dt, kind):
    """The fused digit kernels (byte, 2-byte, 4-byte first passes) raise the status
    bit for a symbol >= sigma anywhere in the text, including the last partial tile."""
    from paper_1702_07578_b200.device import DeviceBuilder

    b = DeviceBuilder()
    n = 3 * 16384 + 123
    g = torch.Generator(device="cuda")
    g.manual_seed(sigma)
    for pos in (0, 20_000, n - 1):
        text = torch.randint(0, sigma, (n,), generator=g, device="cuda", dtype=torch.int64)
        text[pos] = sigma
        with pytest.raises(ValueError):
            b.build(text.to(dt), sigma, kind)


@pytest.mark.parametrize("sigma,kind,hist", [(256, "wm", False), (256, "wt", True), (5, "wm", True),
                                             (1000, "wt", True), (1 << 20, "wm", False)])
def test_pipelined_host_batch_matches_single_builds(sigma, kind, hist):
    """wvlt_build_host_batch (upload / build / download overlapped over three
    streams, double-buffered slots): every build of a ragged queue of texts --
    empty, sub-word, tile-boundary and multi-tile lengths -- equals its own
    oracle build, zeros and histogram included."""
    from paper_1702_07578_b200.device import DeviceBuilder, sym_dtype_for_sigma

    rng = np.random.default_rng(sigma + len(kind))
    dt = sym_dtype_for_sigma(sigma)
    lens = [1_000_003, 0, 63, 16384, 16385, 2_000_000, 777]
    texts = [rng.integers(0, sigma, n).astype(dt) for n in lens]
    b = DeviceBuilder()
    res = b.build_host_batch(texts, sigma, kind, histogram=hist)
    assert len(res) == len(texts)
    for t, (words, zeros, h) in zip(texts, res):
        ww, wz, wh = oracle.build(t, sigma, kind, "pc")
        assert np.array_equal(np.asarray(words).reshape(ww.shape), ww)
        if kind == "wm":
            assert list(zeros) == list(wz)
        if hist:
            assert np.array_equal(h, np.bincount(t, minlength=1 << (sigma - 1).bit_length()).astype(np.int64))
    # a bad symbol in one text of the queue raises the reference's ValueError
    bad = [texts[0].copy(), texts[5].copy()]
    bad[1][12345] = sigma if sigma < np.iinfo(dt).max + 1 else bad[1][12345]
    if sigma < np.iinfo(dt).max + 1:
        with pytest.raises(ValueError):
            b.build_host_batch(bad, sigma, kind)


@pytest.mark.parametrize("sigma,kind", [(256, "wm"), (1000, "wt")])
def test_pageable_host_buffers_are_staged(sigma, kind):
    """wvlt_build_host with pageable (plain numpy) text and output words -- the
    reference API's case -- goes through the staged multi-chunk copies
    (several 32 MiB chunks, odd tail) and equals the device-resident build."""
    from paper_1702_07578_b200.device import DeviceBuilder, sym_dtype_for_sigma

    rng = np.random.default_rng(sigma)
    n = 70_000_003
    text = rng.integers(0, sigma, n).astype(sym_dtype_for_sigma(sigma))
    b = DeviceBuilder()
    words, zeros, _ = b.build_host(text, sigma, kind)
    want = b.build(torch.from_numpy(text).cuda(), sigma, kind)
    assert np.array_equal(words, want.level_words.cpu().numpy().view(np.uint64))
    if kind == "wm":
        assert zeros == [int(z) for z in want.zeros.cpu().tolist()]
    st = wv.build_structure(text[:5_000_001], sigma, kind)
    ref_words, _, _ = oracle.build(text[:5_000_001], sigma, kind, "pc")
    for ell, lv in enumerate(st.levels):
        assert np.array_equal(lv.words, ref_words[ell])


def test_allocation_ledger_of_real_builds(rng):
    """track_allocations around real drop-in builds logs the device workspace
    (positions always; symbols only for wide alphabets; partial_bits for a wide tree)."""
    from paper_1702_07578_b200.construct import track_allocations

    n = 200_001
    for sigma, kind, nsym, partial in [(256, "wm", 0, False), (5, "wt", 0, False), (1 << 16, "wm", 2, False),
                                       (1 << 20, "wt", 2, True)]:
        text = random_text(rng, n, sigma)
        with track_allocations() as log:
            st = wv.build_structure(text, sigma, kind)
        assert wv.dump_structure(st) == ref_dump(text, sigma, kind)
        assert log.position_entries > 0
        assert log.buffers("symbols") == [n] * nsym, (sigma, kind)
        assert bool(log.buffers("partial_bits")) == partial


@pytest.mark.parametrize("kind", ["wt", "wm"])
def test_borders_wider_storage_every_path(kind):
    """Device builds with node borders over storage wider than the alphabet needs
    (u16 / u32 texts with byte or 2-byte alphabets take the generic passes, not
    the fused byte pass) and the byte fast path, all against oracle.borders."""
    from paper_1702_07578_b200.device import DeviceBuilder

    rng = np.random.default_rng(77)
    b = DeviceBuilder()
    for sigma, dt in [(5, torch.uint16), (256, torch.uint32), (1000, torch.uint32), (256, torch.uint8),
                      (70000, torch.uint32), (2, torch.uint8), (3, torch.uint16)]:
        n = 123_457
        text = rng.integers(0, sigma, n).astype(np.int64)
        t = torch.from_numpy(text).to(torch.int32).to(dt).cuda() if dt != torch.uint8 else \
            torch.from_numpy(text.astype(np.uint8)).cuda()
        res = b.build(t, sigma, kind, borders=True, histogram=True)
        w = wv.code_width(sigma)
        hist = oracle.histogram(text, sigma)
        assert np.array_equal(res.hist.cpu().numpy(), hist), (sigma, dt)
        if w >= 2:
            assert np.array_equal(res.borders.cpu().numpy()[: (1 << w) - 2], oracle.borders(hist, w, kind)), (sigma, dt)
        words, zeros, _ = oracle.build(text, sigma, kind, "pc")
        assert np.array_equal(res.level_words.cpu().numpy().view(np.uint64), words), (sigma, dt)


@pytest.mark.parametrize("kind", ["wm", "wt"])
@pytest.mark.parametrize("sigma", [4, 5, 8, 9, 16, 17, 32, 33, 64, 65, 128, 129, 256])
def test_byte_pass_class_extremes(kind, sigma):
    """Inputs that drive the two-levels-per-round byte pass (k8q.cuh) to its
    packed-count limits: whole warp regions (32 runs x 8 symbols) of a single
    2-bit class (a byte field of the exclusive scan at 31 x 8, a warp total of
    256), tiles of one class, alternating classes per run and per symbol, and a
    partial last tile; every width 2..8, against the oracle."""
    rng = np.random.default_rng(sigma * 31 + (kind == "wt"))
    n = 3 * 16384 + 8 * 357 + 5
    top = sigma - 1
    base = np.arange(n)
    texts = {
        "const0": np.zeros(n, np.uint8),
        "const_top": np.full(n, top, np.uint8),
        # runs of 256 symbols (one warp region of one 4-byte region) of one value
        "warp_blocks": (rng.integers(0, sigma, n // 256 + 1).repeat(256)[:n]).astype(np.uint8),
        # each 8-symbol run constant, runs cycling through the values
        "run_cycle": ((base // 8) % sigma).astype(np.uint8),
        # symbol-level alternation of two far-apart values
        "alt": np.where(base % 2 == 0, 0, top).astype(np.uint8),
        # one tile of zeros, one of the top value, then random
        "tiles": np.concatenate([np.zeros(16384, np.uint8), np.full(16384, top, np.uint8),
                                 rng.integers(0, sigma, n - 32768).astype(np.uint8)]),
        # two values that differ only in the lowest bit, in long random runs
        "low_bit": (np.repeat(rng.integers(0, 2, n // 97 + 1), 97)[:n] + (top & ~1)).clip(0, top).astype(np.uint8),
    }
    for name, text in texts.items():
        assert wv.dump_structure(wv.build_structure(text, sigma, kind)) == ref_dump(text, sigma, kind), (sigma, name)


@pytest.mark.parametrize("kind", ["wm", "wt"])
@pytest.mark.parametrize("sigma", [600, 1500, 3000, 5000, 12000, 20000, 1 << 16])
def test_two_byte_pass_every_width(kind, sigma):
    """The fused 2-byte pass at every width W = live bits - 8 (2..8; even widths
    run two levels per round, k16q.cuh): several tiles and a partial one,
    uniform / Zipf / constant / long runs / single-class warp regions, vs the oracle."""
    rng = np.random.default_rng(sigma + (kind == "wt"))
    n = 3 * 16384 + 4 * 333 + 7
    top = sigma - 1
    texts = {
        "uniform": rng.integers(0, sigma, n),
        "zipf": rng.permutation(sigma)[rng.zipf(1.1, n) % sigma],
        "const": np.full(n, top),
        "runs": np.repeat(rng.integers(0, sigma, n // 700 + 1), 700)[:n],
        "blocks256": np.repeat(rng.integers(0, sigma, n // 256 + 1), 256)[:n],
        "alt": np.where(np.arange(n) % 2 == 0, 0, top),
    }
    for name, t in texts.items():
        text = t.astype(np.uint16)
        assert wv.dump_structure(wv.build_structure(text, sigma, kind)) == ref_dump(text, sigma, kind), (sigma, name)
