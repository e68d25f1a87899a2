"""Seeded synthetic inputs for the BASELINE.json configs (benchmark infrastructure).

The paper's corpora are not available; these generators stand in
for them with the configs' shapes, sizes and value distributions.  Texts are
generated on the GPU with torch's seeded Philox generator, in chunks.

  c1  n=2^20  u8  sigma=256  uniform
  c2  n=2^30  u8  sigma=256  Zipf(s=1.1) ranks -> byte values via a seeded permutation
  c3  n=2^30  u8  sigma=4: one order-3 Markov chain, Dirichlet(0.5) transitions
      (generated in parallel segments, exactly; see _markov3_chain);
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
    "c3": "WM n=2^30 u8 sigma=5 one order-3 Markov chain (Dirichlet 0.5 rows, uniform head) + 1% rare symbol",
    "c3s4": "WM n=2^30 u8 sigma=4 one order-3 Markov chain (Dirichlet 0.5 rows, uniform head)",
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


def _markov3_chain(g, n, device, coalesce_steps: int = 256):
    """ONE order-3 Markov chain over {0..3} of n steps: 64 contexts x Dirichlet(0.5)
    transition rows, a uniform initial context (the first 3 symbols), step t
    consuming one uniform draw.

    The chain is computed in 2^14-step segments advanced in lock step.  Pass 1
    runs every segment from all 64 possible entry contexts at once (same draws);
    driven by the same draws the 64 trajectories coalesce within a few dozen
    steps, after which one trajectory per segment is followed (segments that
    have not coalesced after the first 256 steps keep all 64).  That gives each
    segment's exit context as a function of its entry; the entry context of
    every segment then follows sequentially from the chain's head, and pass 2
    replays the same draws from those entries and emits the symbols.  The
    output is exactly the sequential chain (tests/test_workloads.py).
    """
    alpha = torch.full((64, 4), 0.5, dtype=torch.float64, device=device)
    gam = torch._standard_gamma(alpha, generator=g)
    table = torch.cumsum(gam / gam.sum(1, keepdim=True), 1)
    table[:, -1] = 1.0
    seg = 1 << 14
    nseg = max((n + seg - 1) // seg, 1)
    head = int(torch.randint(0, 64, (1,), generator=g, device=device).item())
    state = g.get_state()

    def step(ctx, u):
        sym = (u.view(-1, *([1] * (ctx.dim() - 1)), 1) > table[ctx]).sum(-1).clamp_(max=3)
        return ((ctx << 2) | sym) & 63, sym

    ctx = torch.arange(64, device=device).repeat(nseg, 1)  # [segment, entry context]
    t = 0
    t = min(coalesce_steps, seg)
    for _ in range(t):
        ctx, _ = step(ctx, torch.rand(nseg, generator=g, dtype=torch.float64, device=device))
    coal = (ctx == ctx[:, :1]).all(1)
    single = ctx[:, 0].clone()
    rest = torch.nonzero(~coal).flatten()  # segments still tracked from every entry
    full = ctx[rest]
    for _ in range(t, seg):
        u = torch.rand(nseg, generator=g, dtype=torch.float64, device=device)
        single, _ = step(single, u)
        if rest.numel():
            full, _ = step(full, u[rest])
    exit_of = single.view(-1, 1).expand(nseg, 64).clone()
    if rest.numel():
        exit_of[rest] = full
    exit_of = exit_of.cpu().numpy()
    entries = [0] * nseg
    c = head
    for k in range(nseg):
        entries[k] = c
        c = int(exit_of[k, c])
    g.set_state(state)
    ctx = torch.tensor(entries, device=device)
    buf = torch.empty((nseg, seg), dtype=torch.uint8, device=device)
    for t in range(seg):
        ctx, sym = step(ctx, torch.rand(nseg, generator=g, dtype=torch.float64, device=device))
        buf[:, t] = sym.to(torch.uint8)
    return buf.view(-1)[:n]


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
        out.copy_(_markov3_chain(g, n, device))
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
