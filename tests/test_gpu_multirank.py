"""World > 1 with the real CUDA kernels, R processes sharing ONE GPU.

Only one GPU is available to this project, so the sharded build
(distributed.build_sharded; the reference path it replaces is
construct.build_domain_decomposed, construct.py:437-513) runs as R = 2..4
processes on cuda:0 in a gloo group.  Every process does its local build with
the product kernels (CudaOps), and the merges run on the GPU too:

* transport "nccl": the collectives (size / histogram all_gather, bit-segment
  all_to_all, gather) are staged through host memory (``comm_device="cpu"``,
  the small transport shim), then wvlt_merge_bits shift-merges on the GPU;
* transport "p2p": every rank's local levels are mapped into the other
  processes with CUDA IPC handles (``CudaOps(peer="ipc")``) in place of the
  NVLink symmetric-memory mapping; the merge plan is computed on the device
  from the all-gathered node borders (wvlt_peer_plan) and each owner's words
  are assembled by wvlt_merge_levels_peer reading the other processes' buffers.

This is NOT an NVLink measurement: the ranks share one GPU and one HBM, and
the collectives are host-staged gloo.  It checks that the multi-rank plumbing
(plans, offsets, peer pointers, completion ordering) is right with the real
kernels; rank 0's gathered levels must equal a single build of the whole text
byte for byte, for skewed texts with an empty shard and shard boundaries
inside a word.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _text(n: int, sigma: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    dt = np.uint8 if sigma <= 256 else np.uint16 if sigma <= 65536 else np.uint32
    # Zipf-skewed with a few long runs: groups of very different sizes
    t = (rng.zipf(1.2, n) % sigma).astype(dt)
    t[n // 3: n // 3 + 5000] = sigma - 1
    return t


def _cuts(n: int, world: int, seed: int) -> list[int]:
    rng = np.random.default_rng(seed)
    inner = sorted(int(v) for v in rng.integers(1, n, world - 1))
    inner[0] = 64 * 1000 + 17  # a shard boundary inside a word
    if world > 2:
        inner[1] = inner[0]  # an empty shard
    return [0] + sorted(inner) + [n]


CASES = [(sigma, kind) for sigma in (256, 1 << 16, 1 << 20) for kind in ("wt", "wm")]


def _worker(rank, world, port, transport, n, out_dir):
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1702_07578_b200.device import DeviceBuilder
    from paper_1702_07578_b200.distributed import CudaOps, build_sharded

    ops = CudaOps(peer="ipc")
    results = []
    for ci, (sigma, kind) in enumerate(CASES):
        text = _text(n, sigma, 100 + ci)
        cuts = _cuts(n, world, 200 + ci)
        shard = torch.from_numpy(text[cuts[rank]:cuts[rank + 1]].copy()).cuda()
        for _ in range(2):  # the second build reuses the peer buffers, plan buffers and source table
            res = build_sharded(shard, sigma, kind, ops=ops, gather=True, transport=transport, comm_device="cpu")
        if rank == 0:
            single = DeviceBuilder().build(torch.from_numpy(text).cuda(), sigma, kind)
            ok = torch.equal(res.full_words, single.level_words)
            ok = ok and [int(z) for z in single.zeros.cpu().tolist()] == [int(z) for z in res.zeros]
            results.append((ci, int(bool(ok))))
    if rank == 0:
        np.save(os.path.join(out_dir, "results.npy"), np.array(results, dtype=np.int64))
    torch.cuda.synchronize()
    dist.barrier()
    ops._peer = None  # close the peers' IPC mappings before any producer exits
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_build_real_kernels_one_gpu(world, transport, tmp_path):
    import torch.multiprocessing as mp

    n = 3_000_017
    mp.start_processes(_worker, args=(world, _free_port(), transport, n, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = np.load(tmp_path / "results.npy")
    assert len(res) == len(CASES)
    bad = [CASES[int(ci)] for ci, ok in res if not ok]
    assert not bad, bad


@pytest.mark.parametrize("kind", ["wt", "wm"])
@pytest.mark.parametrize("sigma,world", [(5, 2), (256, 3), (1 << 16, 8), (1 << 20, 8)])
def test_device_plan_kernel_equals_host_restatement(kind, sigma, world):
    """wvlt_peer_plan on the device == plan_from_borders_host (which the CPU tests
    pin to the reference merge order) from the same gathered rows."""
    from paper_1702_07578_b200.bitperm import code_width
    from paper_1702_07578_b200.device import DeviceBuilder
    from paper_1702_07578_b200.distributed import CudaOps, plan_from_borders_host

    n = 400_003
    text = torch.from_numpy(_text(n, sigma, sigma + world)).cuda()
    cuts = _cuts(n, world, world)
    w = code_width(sigma)
    nb = 1 << w
    b = DeviceBuilder()
    rows, borders, ns = [], [], []
    for r in range(world):
        res = b.build(text[cuts[r]:cuts[r + 1]].clone(), sigma, kind, histogram=True, borders=True)
        bd = res.borders[: nb - 2] if w >= 2 else torch.zeros(0, dtype=torch.int64, device="cuda")
        rows.append(torch.cat([res.hist, bd]))
        borders.append(bd.cpu().numpy())
        ns.append(cuts[r + 1] - cuts[r])
    allrows = torch.stack(rows)
    plan = CudaOps().device_plan(allrows, allrows.shape[1], nb, torch.tensor(ns, device="cuda"), world, w, kind)
    want = plan_from_borders_host(borders, ns, kind, w)
    for got, exp in zip(plan, want):
        assert np.array_equal(got.cpu().numpy()[: exp.size], exp)
