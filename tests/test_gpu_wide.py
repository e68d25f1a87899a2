"""Alphabets wider than 24 bits (code widths 25..28, 4-byte symbols).

The reference builds any sigma with a histogram padded to 2^ceil(lg sigma)
entries (construct.py:167-190, levelstats.py:30-47); the device build takes
code widths up to WVLT_MAX_WIDTH = 28: K = 4 passes over the 4-byte symbols
until 24 live bits remain, then the fused 4-byte / 2-byte / byte stages, the
tree by the group recurrence over 2^w groups (nearly all empty at these text
sizes: the merge's task search has to skip them, not walk them).  Compared
word for word with the oracle's pc builder, with histogram and node borders at
w = 25.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402


@pytest.mark.parametrize("kind", ["wm", "wt"])
@pytest.mark.parametrize("w", [25, 26, 28])
def test_code_widths_above_24(kind, w):
    rng = np.random.default_rng(w * 2 + (kind == "wm"))
    b = DeviceBuilder()
    for sigma in (1 << w, (1 << (w - 1)) + 12345):
        n = int(rng.integers(100_000, 400_000))
        host = np.minimum(np.floor(np.exp2(rng.random(n) * np.log2(sigma))), sigma - 1).astype(np.uint32)  # log-uniform
        host[::7] = rng.integers(0, sigma, host[::7].size)
        host[-1] = sigma - 1
        extras = w == 25
        res = b.build(torch.from_numpy(host).cuda(), sigma, kind, borders=extras, histogram=extras)
        words, zeros, _ = res.to_host()
        ow, oz, _ = oracle.build(host, sigma, kind, "pc")
        assert np.array_equal(words, ow), (w, kind, sigma)
        if kind == "wm":
            assert zeros == oz
        if extras:
            import paper_1702_07578_b200 as wv

            st = wv.build_structure(host, sigma, kind)  # the drop-in call on the host array
            assert wv.dump_structure(st) == oracle.dump(kind, n, sigma, ow, oz)
            hist = oracle.histogram(host, sigma)
            assert np.array_equal(res.hist.cpu().numpy(), hist)
            assert np.array_equal(res.borders.cpu().numpy()[: (1 << w) - 2], oracle.borders(hist, w, kind))
        del res
        torch.cuda.empty_cache()


def test_width_above_the_limit_is_rejected():
    b = DeviceBuilder()
    t = torch.zeros(100, dtype=torch.uint32, device="cuda")
    with pytest.raises(ValueError):
        b.build(t, (1 << 28) + 1, "wm")
