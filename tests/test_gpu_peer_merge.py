"""The multi-GPU merge over peer memory (wvlt_merge_levels_peer) on one GPU.

One GPU cannot host several ranks, so the kernel is checked with every
"peer" buffer on the same device: R local builds of R shards, their level
addresses handed to the kernel exactly as the p2p transport hands it the
peer-mapped symmetric-memory addresses, and the owners' word ranges
reassembled must equal the single build.  The p2p transport itself
(symmetric-memory rendezvous, plan, merge, completion collective) runs end to
end in a one-rank NCCL group.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1702_07578_b200.bitperm import code_width  # noqa: E402
from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402
from paper_1702_07578_b200.distributed import CudaOps, exchange_plan, peer_plan_arrays  # noqa: E402


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("sigma,world,n", [(5, 2, 100_003), (256, 4, 1 << 20), (1000, 3, 300_001),
                                           (1 << 16, 8, 1 << 21), (1 << 20, 5, 500_000)])
def test_peer_merge_kernel_reassembles_the_single_build(kind, sigma, world, n):
    g = torch.Generator(device="cuda")
    g.manual_seed(sigma + world)
    dt = torch.uint8 if sigma <= 256 else torch.uint16 if sigma <= 65536 else torch.uint32
    text = torch.randint(0, sigma, (n,), generator=g, device="cuda", dtype=torch.int64).to(dt)
    rng = np.random.default_rng(world)
    cuts = [0] + sorted(rng.choice(np.arange(1, n), world - 1, replace=False).tolist()) + [n]
    width = code_width(sigma)
    b = DeviceBuilder()
    locs, hists = [], []
    for r in range(world):
        res = b.build(text[cuts[r]:cuts[r + 1]].clone(), sigma, kind, histogram=True)
        locs.append(res.level_words)
        hists.append(res.hist.cpu().numpy())
    lns = [cuts[r + 1] - cuts[r] for r in range(world)]
    ranges, plans = exchange_plan(np.stack(hists), kind, width, n, lns, world)
    want = b.build(text, sigma, kind).level_words
    ops = CudaOps()
    for owner, (w0, w1) in enumerate(ranges):
        level_src = np.array([[locs[r].data_ptr() + 8 * ell * locs[r].shape[1] for r in range(world)]
                              for ell in range(width)], dtype=np.int64)
        owned = torch.full((width, w1 - w0), -1, dtype=torch.int64, device="cuda")
        ops.merge_peer(owned, w0, w1, n, peer_plan_arrays(plans, owner, width), level_src, world)
        assert torch.equal(owned, want[:, w0:w1]), owner


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_p2p_transport_one_rank_group():
    import torch.distributed as dist

    from paper_1702_07578_b200.distributed import build_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = torch.Generator(device="cuda")
        g.manual_seed(3)
        for sigma, kind in ((256, "wm"), (1000, "wt")):
            dt = torch.uint8 if sigma <= 256 else torch.uint16
            text = torch.randint(0, sigma, (333_333,), generator=g, device="cuda", dtype=torch.int64).to(dt)
            res = build_sharded(text, sigma, kind, transport="p2p", gather=True)
            want = DeviceBuilder().build(text, sigma, kind)
            assert torch.equal(res.full_words, want.level_words)
            assert res.zeros == [int(z) for z in want.zeros.cpu().tolist()] or kind == "wt"
        # an out-of-range symbol raises the reference's ValueError on every rank
        # (the range flag travels with the histogram all_gather)
        for transport in ("p2p", "nccl"):
            bad = torch.full((100_000,), 3, dtype=torch.uint8, device="cuda")
            bad[77_777] = 200
            with pytest.raises(ValueError):
                build_sharded(bad, 100, "wm", transport=transport)
    finally:
        dist.destroy_process_group()
