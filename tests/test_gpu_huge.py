"""Texts around and past 2^32 symbols, where positions stop fitting 32 bits.

The fused byte pass and the fused wide-alphabet stages carry 32-bit tile-local
and global positions and are only eligible below 2^32 - 64 symbols
(k8_eligible, make_plan); longer texts take the K = 4 passes with 64-bit
positions.  Both sides of that switch are compared word for word with the
oracle's ps builder (construct.py:322-387) on all host cores -- the reference
itself builds any n (test_construct.py:205-226 is its own large-n check).
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

from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402


@pytest.mark.parametrize("sigma,kind,dt,n", [
    (256, "wm", "uint8", (1 << 32) + 4099),   # past the limit: K = 4 byte passes
    (5, "wt", "uint8", (1 << 32) - 64),       # the first length the fused byte pass refuses
    (5, "wm", "uint8", (1 << 32) - 65),       # the last length it takes
    (1000, "wm", "uint16", (1 << 32) + 77),   # two-byte symbols past the limit
])
def test_build_around_2_pow_32_symbols(sigma, kind, dt, n):
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * (1 << 30):  # pragma: no cover
        pytest.skip("needs ~40 GB of device memory")
    try:
        import psutil

        if psutil.virtual_memory().available < 48 * (1 << 30):  # pragma: no cover
            pytest.skip("needs ~48 GB of host memory for the oracle")
    except ImportError:  # pragma: no cover
        pass
    tdt = getattr(torch, dt)
    g = torch.Generator(device="cuda")
    g.manual_seed(sigma + n % 1000)
    text = torch.empty(n, dtype=tdt, device="cuda")
    step = 1 << 28
    for i in range(0, n, step):
        m = min(step, n - i)
        r = torch.rand(m, generator=g, device="cuda")
        text[i:i + m] = (r * r * sigma).to(torch.int32).clamp_(max=sigma - 1).to(tdt)  # skewed towards small values
    res = DeviceBuilder().build(text, sigma, kind)
    host = text.cpu().numpy()
    del text
    ow, oz, _ = oracle.build(host, sigma, kind, "ps", threads=os.cpu_count() or 1)
    for level in range(res.width):
        assert np.array_equal(res.level_words[level].cpu().numpy().view(np.uint64), ow[level]), level
    if kind == "wm":
        assert [int(z) for z in res.zeros.cpu().tolist()] == oz
