"""Adversarial histogram tests for the wide-alphabet histogram kernel.

``hist_generic_kernel`` keeps two bins per shared 32-bit word as 16-bit
counters and carries wraps into the global histogram from each atomic's old
value.  The texts here make the two bins of one word both hot (alternating
2k / 2k+1, hundreds of thousands of increments of each per CTA), so low-half
wraps and high-half increments interleave constantly; every histogram must
equal ``np.bincount`` exactly (levelstats.symbol_histogram, levelstats.py:30-47;
_kernels.hist_and_msb_bits, _kernels.py:23-36).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import workloads  # noqa: E402
from paper_1702_07578_b200 import _lib  # noqa: E402
from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402


def device_histogram(text: "torch.Tensor", sigma: int) -> np.ndarray:
    """wvlt_histogram through the C ABI on a device text."""
    w = max(sigma - 1, 0).bit_length()
    hist = torch.zeros(1 << w, dtype=torch.int64, device=text.device)
    status = torch.zeros(1, dtype=torch.int32, device=text.device)
    rc = _lib.load().wvlt_histogram(text.data_ptr(), text.element_size(), int(text.numel()), int(sigma),
                                    hist.data_ptr(), status.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    assert int(status.item()) == 0
    return hist.cpu().numpy()


def bincount(text: "torch.Tensor", nbins: int) -> np.ndarray:
    signed = {torch.uint8: torch.uint8, torch.uint16: torch.int16, torch.uint32: torch.int32}[text.dtype]
    mask = (1 << (8 * text.element_size())) - 1
    v = text.view(signed).to(torch.int64) & mask
    return torch.bincount(v, minlength=nbins).cpu().numpy()


def alternating_u16(n: int, k: int, seed: int, mix: float = 0.0) -> "torch.Tensor":
    """2k, 2k+1, 2k, 2k+1, ...; with ``mix`` > 0 a fraction of positions is
    redrawn uniformly from {2k, 2k+1} (unequal, randomly interleaved halves)."""
    i = torch.arange(n, device="cuda", dtype=torch.int64)
    v = 2 * k + (i & 1)
    if mix:
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)
        flip = torch.rand(n, generator=g, device="cuda") < mix
        v = torch.where(flip, 2 * k + torch.randint(0, 2, (n,), generator=g, device="cuda"), v)
    return v.to(torch.int32).to(torch.uint16)


@pytest.mark.parametrize("k,mix", [(0, 0.0), (0, 0.3), (12345, 0.0), (32767, 0.5)])
def test_wvlt_histogram_hot_pair_u16(k, mix):
    n = 1 << 28
    text = alternating_u16(n, k, seed=k + 1, mix=mix)
    want = bincount(text, 1 << 16)
    got = device_histogram(text, 1 << 16)
    assert np.array_equal(got, want)
    del text
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kind", ["wm", "wt"])
def test_build_histogram_hot_pair_u16(kind):
    """histogram=True builds of a 2-byte text (the tables and zero counts use it)."""
    n = 1 << 28
    text = alternating_u16(n, 0, seed=5, mix=0.1)
    want = bincount(text, 1 << 16)
    res = DeviceBuilder().build(text, 1 << 16, kind, histogram=True)
    assert np.array_equal(res.hist.cpu().numpy(), want)
    h = want.copy()
    zeros = []
    for _ in range(16):
        zeros.append(int(h[0::2].sum()))
        h = h[0::2] + h[1::2]
    assert [int(z) for z in res.zeros.cpu().tolist()] == zeros[::-1]
    del text, res
    torch.cuda.empty_cache()


def test_u16_text_small_alphabet_hot_pair():
    """A uint16 text with sigma <= 256 takes the generic histogram (wide symbols)."""
    n = (1 << 27) + 3
    text = (torch.arange(n, device="cuda", dtype=torch.int64) & 1).to(torch.int32).to(torch.uint16)
    want = bincount(text, 2)
    assert np.array_equal(device_histogram(text, 2), want)
    for kind in ("wt", "wm"):
        res = DeviceBuilder().build(text, 2, kind, histogram=True)
        assert np.array_equal(res.hist.cpu().numpy(), want)


def test_c5_histogram_log_uniform():
    """c5's log-uniform u32 text: bins 0 and 1 (one shared word) are the two hottest."""
    torch.cuda.empty_cache()
    text = workloads.generate("c5")
    sigma = workloads.CONFIGS["c5"]["sigma"]
    want = bincount(text, sigma)
    assert want[0] > (1 << 26) and want[1] > (1 << 25)
    assert np.array_equal(device_histogram(text, sigma), want)
    res = DeviceBuilder().build(text, sigma, "wm", histogram=True)
    assert np.array_equal(res.hist.cpu().numpy(), want)
    del text, res
    torch.cuda.empty_cache()
