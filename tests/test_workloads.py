"""The synthetic config generators (benchmark / test infrastructure, CPU)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import workloads


@pytest.mark.parametrize("coalesce_steps", [256, 1, 0])
def test_markov3_chain_is_one_sequential_chain(coalesce_steps):
    """The segment-parallel generator equals the chain run step by step with the
    same draws (one order-3 Markov chain, Dirichlet(0.5) rows), also
    when segments are still followed from every entry context (few or no
    coalescing steps)."""
    n = (1 << 14) * 3 + 77
    g = torch.Generator()
    g.manual_seed(3)
    out = workloads._markov3_chain(g, n, "cpu", coalesce_steps).numpy()
    g = torch.Generator()
    g.manual_seed(3)
    alpha = torch.full((64, 4), 0.5, dtype=torch.float64)
    gam = torch._standard_gamma(alpha, generator=g)
    table = torch.cumsum(gam / gam.sum(1, keepdim=True), 1)
    table[:, -1] = 1.0
    head = int(torch.randint(0, 64, (1,), generator=g).item())
    nseg = (n + (1 << 14) - 1) >> 14
    draws = torch.stack([torch.rand(nseg, generator=g, dtype=torch.float64) for _ in range(1 << 14)], 1)
    u = draws.reshape(-1)[:n].numpy()
    rows = table.numpy()
    ref = np.empty(n, dtype=np.uint8)
    c = head
    for i in range(n):
        s = min(int((u[i] > rows[c]).sum()), 3)
        ref[i] = s
        c = ((c << 2) | s) & 63
    assert np.array_equal(out, ref)


def test_generators_shapes_and_ranges():
    for name in ("c1", "c3", "c3s4", "c4", "c5"):
        cfg = workloads.CONFIGS[name]
        t = workloads.generate(name, device="cpu", n=(1 << 15) + 5)
        assert t.dtype == cfg["dtype"] and t.numel() == (1 << 15) + 5
        v = t.to(torch.int64) & ((1 << (8 * t.element_size())) - 1)
        assert int(v.min()) >= 0 and int(v.max()) < cfg["sigma"]
