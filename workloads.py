"""Seeded synthetic inputs for the BASELINE.json configs (benchmark infrastructure).

The paper's corpora are not available; these generators stand in
for them with the configs' shapes, sizes and value distributions.  Texts are
generated on the GPU with torch's seeded Philox generator, in chunks.

  c1  n=2^20  u8  sigma=256  uniform
  c2  n=2^30  u8  sigma=256  Zipf(s=1.1) ranks -> byte values via a seeded permutation
  c3  n=2^30  u8  sigma=4 order-3 Markov chain, Dirichlet(0.5) transitions;
      variant sigma=5 replaces 1% of positions by the rare symbol 4
  c4  n=2^29  u16 sigma=2^16: 50% Zipf(s=1.0) over all values, 50% uniform over a
      random 4096-value subset
  c5  n=2^31  u32 sigma=2^20: floor(2^(20 U)) - 1, U uniform (log-uniform values)
"""

from __future__ import annotations

import torch

CONFIGS = {
    "c1": dict(n=1 << 20, sigma=256, dtype=torch.uint8, kind="wt"),
    "c2": dict(n=1 << 30, sigma=256, dtype=torch.uint8, kind="wm"),
    "c3": dict(n=1 << 30, sigma=5, dtype=torch.uint8, kind="wm"),
    "c3s4": dict(n=1 << 30, sigma=4, dtype=torch.uint8, kind="wm"),
    "c4": dict(n=1 << 29, sigma=1 << 16, dtype=torch.uint16, kind="wm"),
    "c5": dict(n=1 << 31, sigma=1 << 20, dtype=torch.uint32, kind="wm"),
}

DESCRIPTIONS = {
    "c1": "WT n=2^20 u8 sigma=256 uniform",
    "c2": "WM n=2^30 u8 sigma=256 Zipf(1.1) ranks via seeded permutation",
    "c3": "WM n=2^30 u8 sigma=5 order-3 Markov (Dirichlet 0.5) + 1% rare symbol",
    "c3s4": "WM n=2^30 u8 sigma=4 order-3 Markov (Dirichlet 0.5)",
    "c4": "WM n=2^29 u16 sigma=2^16 50% Zipf(1.0) + 50% uniform over 4096-subset",
    "c5": "WM n=2^31 u32 sigma=2^20 log-uniform",
}

SEED = 0x574C54
CHUNK = 1 << 26


def _zipf_ranks(g, n, k, s, device):
    ranks = torch.arange(1, k + 1, dtype=torch.float64, device=device)
    p = ranks.pow(-s)
    cdf = torch.cumsum(p / p.sum(), 0)
    cdf[-1] = 1.0
    u = torch.rand(n, generator=g, dtype=torch.float64, device=device)
    return torch.searchsorted(cdf, u).clamp_(max=k - 1)


def generate(name: str, device="cuda", n: int | None = None, seed: int | None = None) -> torch.Tensor:
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    seed = SEED + list(CONFIGS).index(name) if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty(n, dtype=cfg["dtype"], device=device)
    sigma = cfg["sigma"]
    if name == "c1":
        for i in range(0, n, CHUNK):
            m = min(CHUNK, n - i)
            out[i : i + m] = torch.randint(0, 256, (m,), generator=g, device=device, dtype=torch.int32).to(torch.uint8)
    elif name == "c2":
        perm = torch.randperm(256, generator=g, device=device)
        for i in range(0, n, CHUNK):
            m = min(CHUNK, n - i)
            out[i : i + m] = perm[_zipf_ranks(g, m, 256, 1.1, device)].to(torch.uint8)
    elif name in ("c3", "c3s4"):
        # 64 contexts x Dirichlet(0.5) rows; independent chain segments of 2^14
        # steps advanced in lock step (segment heads drawn uniformly)
        alpha = torch.full((64, 4), 0.5, dtype=torch.float64, device=device)
        gam = torch._standard_gamma(alpha, generator=g)
        table = torch.cumsum(gam / gam.sum(1, keepdim=True), 1)
        table[:, -1] = 1.0
        seg = 1 << 14
        nseg = (n + seg - 1) // seg
        ctx = torch.randint(0, 64, (nseg,), generator=g, device=device)
        buf = torch.empty((nseg, seg), dtype=torch.uint8, device=device)
        for t in range(seg):
            u = torch.rand(nseg, generator=g, dtype=torch.float64, device=device)
            sym = (u.unsqueeze(1) > table[ctx]).sum(1).clamp_(max=3)
            buf[:, t] = sym.to(torch.uint8)
            ctx = ((ctx << 2) | sym) & 63
        out.copy_(buf.view(-1)[:n])
        if name == "c3":
            for i in range(0, n, CHUNK):
                m = min(CHUNK, n - i)
                rare = torch.rand(m, generator=g, device=device) < 0.01
                out[i : i + m].masked_fill_(rare, 4)
    elif name == "c4":
        perm = torch.randperm(1 << 16, generator=g, device=device)
        subset = torch.randperm(1 << 16, generator=g, device=device)[:4096]
        for i in range(0, n, CHUNK):
            m = min(CHUNK, n - i)
            z = perm[_zipf_ranks(g, m, 1 << 16, 1.0, device)]
            uni = subset[torch.randint(0, 4096, (m,), generator=g, device=device)]
            coin = torch.rand(m, generator=g, device=device) < 0.5
            out[i : i + m] = torch.where(coin, z, uni).to(torch.int32).to(torch.uint16)
    elif name == "c5":
        for i in range(0, n, CHUNK):
            m = min(CHUNK, n - i)
            u = torch.rand(m, generator=g, dtype=torch.float64, device=device)
            v = torch.floor(torch.exp2(20.0 * u)) - 1
            out[i : i + m] = v.clamp_(0, sigma - 1).to(torch.int64).to(torch.uint32)
    else:
        raise KeyError(name)
    return out
