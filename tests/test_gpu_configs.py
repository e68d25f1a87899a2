"""Full-size BASELINE.json configs on the GPU.

Every config (c1, c2, c3, c3 sigma=4, c4, c5), as WT and as WM, is compared
byte for byte with the oracle's ps builder (the restatement of
construct.py:322-387, pinned to the reference's golden vectors) run on all
host cores at full size -- the analogue of the reference's own all-builders
agreement check at 10^8 symbols (test_construct.py:205-226).  c5's 20 levels
are compared one level at a time to bound host memory.

The builds are also checked by size-independent properties:

* decode: ``access(i)`` computed from the built levels with the reference's
  query algorithms (WT: structures.py:107-125, WM: structures.py:201-215),
  vectorised in torch over 2^16 random positions, must return ``text[i]``;
* zero counts: Z[l] = rank0(level l, n) = zeros_from_histogram of the folded
  histogram (test_acceptance.py:166-181);
* popcount of level l = number of symbols with code bit l set.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import workloads  # noqa: E402
from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402

M1, M2, M4, M8 = 0x5555555555555555, 0x3333333333333333, 0x0F0F0F0F0F0F0F0F, 0x0101010101010101


def popcount64(x: "torch.Tensor") -> "torch.Tensor":
    """SWAR popcount of int64 words (bit patterns), as int64."""
    def c(v):
        return v - (1 << 64) if v >= (1 << 63) else v

    x = x - ((x >> 1) & c(M1))
    x = (x & c(M2)) + ((x >> 2) & c(M2))
    x = (x + (x >> 4)) & c(M4)
    return ((x * c(M8)) >> 56) & 0xFF


class Ranker:
    """rank1(i) over one level's words: cumulative popcount per word."""

    def __init__(self, words: "torch.Tensor"):
        pc = popcount64(words)
        self.cum = torch.cat([torch.zeros(1, dtype=torch.int64, device=words.device), torch.cumsum(pc, 0)])
        self.words = words

    def rank1(self, i):
        w = i >> 6
        r = i & 63
        word = self.words[torch.clamp(w, max=self.words.numel() - 1)]
        mask = torch.where(r > 0, (torch.ones_like(r) << r) - 1, torch.zeros_like(r))
        part = popcount64(word & mask)
        return self.cum[w] + torch.where(r > 0, part, torch.zeros_like(part))

    def bit(self, i):
        return (self.words[i >> 6] >> (i & 63)) & 1


def decode(kind, levels, zeros, n, width, pos):
    rk = [Ranker(levels[l]) for l in range(width)]
    value = torch.zeros_like(pos)
    p = pos.clone()
    if kind == "wm":
        for l in range(width):
            b = rk[l].bit(p)
            r1 = rk[l].rank1(p)
            value = (value << 1) | b
            p = torch.where(b == 1, zeros[l] + r1, p - r1)
        return value
    s = torch.zeros_like(pos)
    e = torch.full_like(pos, n)
    for l in range(width):
        R = rk[l]
        rs1, re1, rp1 = R.rank1(s), R.rank1(e), R.rank1(p)
        z = (e - re1) - (s - rs1)
        b = R.bit(p)
        value = (value << 1) | b
        one = b == 1
        p_one = s + z + (rp1 - rs1)
        p_zero = s + ((p - rp1) - (s - rs1))
        p = torch.where(one, p_one, p_zero)
        s_new = torch.where(one, s + z, s)
        e = torch.where(one, e, s + z)
        s = s_new
    return value


@pytest.mark.parametrize("config,kind", [("c2", "wm"), ("c2", "wt"), ("c3", "wm"), ("c3", "wt"), ("c3s4", "wt"),
                                         ("c4", "wm"), ("c4", "wt"), ("c5", "wm"), ("c5", "wt")])
def test_config_full_size_properties(config, kind):
    cfg = workloads.CONFIGS[config]
    n, sigma = cfg["n"], cfg["sigma"]
    torch.cuda.empty_cache()
    text = workloads.generate(config)
    b = DeviceBuilder()
    # histogram-free build (the WM default), checked against a build that also
    # returns the histogram: identical levels and zero counts
    res = b.build(text, sigma, kind)
    width = res.width
    levels = res.level_words
    full = b.build(text, sigma, kind, histogram=True)
    assert torch.equal(full.level_words, levels)
    assert torch.equal(full.zeros, res.zeros)
    # zero counts vs the histogram (and vs rank0 of each level)
    hist = full.hist.cpu().numpy()
    del full
    h = hist.copy()
    exp_zeros = []
    for l in range(width - 1, -1, -1):
        exp_zeros.append(int(h[0::2].sum()))
        h = h[0::2] + h[1::2]
    exp_zeros = exp_zeros[::-1]
    zeros = [int(z) for z in res.zeros.cpu().tolist()]
    assert zeros == exp_zeros
    for l in range(width):
        assert int(popcount64(levels[l]).sum()) == n - zeros[l], l
    # decode sampled positions
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    pos = torch.randint(0, n, (1 << 16,), generator=g, device="cuda", dtype=torch.int64)
    pos[:4] = torch.tensor([0, 1, n - 2, n - 1], device="cuda")
    got = decode(kind, levels, torch.tensor(zeros, device="cuda"), n, width, pos)
    signed = {torch.uint8: torch.uint8, torch.uint16: torch.int16, torch.uint32: torch.int32}[text.dtype]
    want = text.view(signed)[pos].to(torch.int64) & ((1 << (8 * text.element_size())) - 1)
    assert torch.equal(got, want)
    del res, text, levels
    torch.cuda.empty_cache()


@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c3s4", "c4", "c5"])
def test_config_bytes_vs_oracle_ps(config):
    """Default build (the WM one histogram-free) byte for byte vs oracle ps; the
    build with node borders requested gives the same levels and the borders of
    the oracle's histogram (oracle.borders, the interval_starts /
    interval_start_table restatement)."""
    cfg = workloads.CONFIGS[config]
    torch.cuda.empty_cache()
    text = workloads.generate(config)
    host = text.cpu().numpy()
    threads = os.cpu_count() or 1
    hist = oracle.histogram(host, cfg["sigma"])
    b = DeviceBuilder()
    for kind in ("wm", "wt"):
        res = b.build(text, cfg["sigma"], kind)
        ow, oz, _ = oracle.build(host, cfg["sigma"], kind, "ps", threads)
        assert ow.shape == tuple(res.level_words.shape)
        for ell in range(res.width):
            got = res.level_words[ell].cpu().numpy().view(np.uint64)
            bad = np.flatnonzero(got != ow[ell])
            assert bad.size == 0, (config, kind, ell, int(bad[0]) if bad.size else None, bad.size)
        if kind == "wm":
            assert [int(z) for z in res.zeros.cpu().tolist()] == oz
        del ow
        full = b.build(text, cfg["sigma"], kind, borders=True, histogram=True)
        assert torch.equal(full.level_words, res.level_words), (config, kind)
        assert torch.equal(full.zeros, res.zeros)
        assert np.array_equal(full.hist.cpu().numpy(), hist)
        w = res.width
        assert np.array_equal(full.borders.cpu().numpy()[: (1 << w) - 2], oracle.borders(hist, w, kind))
        del res, full
    del text, host
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kind", ["wm", "wt"])
def test_byte_text_beyond_2_31_symbols(kind):
    """The single fused pass keeps 32-bit bit positions (n < 2^32 - 64): a c2-like
    text of 2^31 + 12345 symbols (past every signed 32-bit boundary), checked by
    decode, zero counts and popcounts."""
    n = (1 << 31) + 12345
    torch.cuda.empty_cache()
    text = workloads.generate("c2", n=n)
    b = DeviceBuilder()
    res = b.build(text, 256, kind, histogram=True)
    levels = res.level_words
    hist = res.hist.cpu().numpy()
    assert int(hist.sum()) == n
    h = hist.copy()
    exp_zeros = []
    for _ in range(8):
        exp_zeros.append(int(h[0::2].sum()))
        h = h[0::2] + h[1::2]
    exp_zeros = exp_zeros[::-1]
    assert [int(z) for z in res.zeros.cpu().tolist()] == exp_zeros
    for ell in range(8):
        assert int(popcount64(levels[ell]).sum()) == n - exp_zeros[ell], ell
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    pos = torch.randint(0, n, (1 << 16,), generator=g, device="cuda", dtype=torch.int64)
    pos[:4] = torch.tensor([0, (1 << 31) - 1, 1 << 31, n - 1], device="cuda")
    got = decode(kind, levels, res.zeros, n, 8, pos)
    assert torch.equal(got, text[pos].to(torch.int64))
    del res, text, levels
    torch.cuda.empty_cache()
