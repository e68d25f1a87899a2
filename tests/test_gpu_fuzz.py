"""Seeded random sweep of the device build against the oracle.

compute-sanitizer is not available on the GPU pool, so a wrong address has to
show up as a wrong bit: every case draws its own length (around word, tile and
multi-tile boundaries), alphabet (every code width 1..20, at and off powers of
two), storage dtype (at least as wide as the code), symbol distribution, pointer
misalignment, structure kind and optional outputs (histogram, node borders),
builds on the GPU through the C ABI and must equal the oracle's pc builder
(construct.py:292-319) word for word, with its zero counts, histogram
(levelstats.py:30-47) and borders (levelstats.py:58-73, wt2wm.py:55-78).
Canary words around the level buffer must stay untouched.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_07578_b200.bitperm import code_width  # noqa: E402
from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402

CANARY = -0x0123456789ABCDEF
PAD = 64  # canary words on each side of the level buffer


def _length(rng) -> int:
    kind = rng.integers(0, 6)
    if kind == 0:
        return int(rng.integers(1, 200))
    if kind == 1:  # around a 64-bit word / 512-bit block
        return int(rng.choice([64, 512, 4096]) * rng.integers(1, 20) + rng.integers(-2, 3))
    if kind == 2:  # around the 8192 / 16384-symbol tiles
        return int(rng.choice([8192, 16384]) * rng.integers(1, 9) + rng.integers(-65, 66))
    if kind == 3:
        return int(rng.integers(200, 70_000))
    return int(rng.integers(70_000, 400_000))


def _sigma(rng) -> int:
    w = int(rng.integers(1, 21))
    choice = rng.integers(0, 4)
    if choice == 0:
        return 1 << w
    if choice == 1:
        return (1 << (w - 1)) + 1
    return int(rng.integers((1 << (w - 1)) + 1, (1 << w) + 1))


def _text(rng, n: int, sigma: int) -> np.ndarray:
    d = rng.integers(0, 7)
    if d == 0:
        t = rng.integers(0, sigma, n)
    elif d == 1:  # heavy hitters
        t = rng.permutation(sigma)[np.minimum(rng.zipf(1.2, n) - 1, sigma - 1)]
    elif d == 2:  # long runs (tiles inside one node, tiles spanning many)
        k = int(rng.integers(1, 60))
        t = np.repeat(rng.integers(0, sigma, k), rng.integers(1, max(2, 2 * n // k), k))[:n]
        t = np.concatenate([t, rng.integers(0, sigma, n - t.size)])
    elif d == 3:
        t = np.sort(rng.integers(0, sigma, n))
    elif d == 4:  # two or three symbols only, the extremes among them
        t = rng.choice(np.unique([0, sigma - 1, int(rng.integers(0, sigma))]), n)
    elif d == 5:  # alternating neighbours (2k, 2k + 1): every split separates adjacent symbols
        b = int(rng.integers(0, max(sigma // 2, 1))) * 2
        t = np.minimum(b + (np.arange(n) & 1), sigma - 1)
    else:  # log-uniform
        t = np.minimum(np.floor(np.exp2(rng.random(n) * np.log2(sigma))) - 1, sigma - 1).clip(0)
    return np.asarray(t, dtype=np.int64)


@pytest.mark.parametrize("seed", range(12))
def test_random_builds_equal_the_oracle(seed):
    rng = np.random.default_rng(0xF00D + seed)
    b = DeviceBuilder()
    for case in range(50):
        n, sigma = _length(rng), _sigma(rng)
        w = code_width(sigma)
        kind = "wm" if rng.integers(0, 2) else "wt"
        dts = [d for d, bits in ((np.uint8, 8), (np.uint16, 16), (np.uint32, 32)) if bits >= w]
        dt = dts[int(rng.integers(0, len(dts)))]
        host = _text(rng, n, sigma).astype(dt)
        off = int(rng.integers(0, 4)) if rng.integers(0, 3) == 0 else 0  # elements of pointer misalignment
        dev = torch.from_numpy(np.concatenate([np.zeros(off, dt), host])).cuda()[off:]
        want_hist, want_borders = bool(rng.integers(0, 2)), bool(rng.integers(0, 2)) and w >= 2
        tag = (seed, case, n, sigma, kind, np.dtype(dt).name, off, want_hist, want_borders)

        nwords = (n + 63) >> 6
        guard = torch.full((2 * PAD + w * nwords,), CANARY, dtype=torch.int64, device="cuda")
        lw, zeros, hist, bd, status = b.alloc_outputs(n, sigma, borders=want_borders)
        lw = guard[PAD:PAD + w * nwords].view(w, nwords)
        res = b.build(dev, sigma, kind, histogram=want_hist, borders=want_borders,
                      outputs=(lw, zeros, hist, bd, status))
        words, zs, _ = res.to_host()
        ow, oz, _ = oracle.build(host, sigma, kind, "pc")
        assert np.array_equal(words, ow), tag
        if kind == "wm":
            assert zs == oz, tag
        g = guard.cpu().numpy()
        assert (g[:PAD] == CANARY).all() and (g[PAD + w * nwords:] == CANARY).all(), tag
        if want_hist:
            assert np.array_equal(res.hist.cpu().numpy()[: 1 << w], oracle.histogram(host, sigma)), tag
        if want_borders:
            assert np.array_equal(res.borders.cpu().numpy()[: (1 << w) - 2],
                                  oracle.borders(oracle.histogram(host, sigma), w, kind)), tag
