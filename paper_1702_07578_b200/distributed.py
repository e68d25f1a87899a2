"""Multi-GPU construction: the text is sharded by position across ranks.

The reference's domain decomposition (construct.build_domain_decomposed,
construct.py:437-513) builds one partial structure per text slice and then
merges every level by moving whole intervals (_merge_plan, construct.py:516-543;
gather_bits, _kernels.py:196-232).  Here the slices are the ranks of a
torch.distributed process group (one process per GPU, NCCL over NVLink):

1. every rank builds the complete local WT/WM of its shard on its GPU
   (no communication);
2. one all_gather of the per-rank symbol histograms (2^w int64 each) gives
   every rank the merge plan of every level: prefix groups in interval order
   (numeric for WT, bit-reversed for WM, construct.py:498), ranks in text order
   inside each group -- the interleaved (prefix, core) order of
   levelstats.interleaved_starts (levelstats.py:76-94) with cores -> ranks;
3. one all_to_all_single moves, for every level, the bit segments each rank
   needs to the rank owning the destination words (word ranges split like
   construct._word_ranges, construct.py:214-217, so every rank owns 1/R of
   every level);
4. every rank shift-merges its word range of every level (wvlt_merge_bits).

The result is bit-identical to the single-GPU build (the reference guarantees
the same for any slice count, test_construct.py:43-51).  The host-side plan
and exchange logic is backend-agnostic so the CPU tests can run it on the
gloo backend with the oracle standing in for the device kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .bitperm import bit_reversal_permutation, code_width


@dataclass
class ShardedResult:
    """This rank's share of a sharded build."""

    n: int                  # global text length
    sigma: int
    kind: str
    width: int
    word_lo: int            # owned global word range [word_lo, word_hi) of every level
    word_hi: int
    level_words: object     # tensor int64 [width, word_hi - word_lo] (uint64 bit patterns)
    zeros: list             # global per-level zero counts
    hist: np.ndarray        # global symbol histogram (2^width)


def word_ranges(total_words: int, world: int) -> list[tuple[int, int]]:
    """construct._word_ranges (construct.py:214-217)."""
    cuts = [(total_words * c) // world for c in range(world + 1)]
    return [(cuts[c], cuts[c + 1]) for c in range(world)]


def fold_to(hist: np.ndarray, width: int, ell: int) -> np.ndarray:
    """Counts of the ell-bit prefixes (fold_pairs applied width-ell times, _kernels.py:45-49)."""
    h = np.asarray(hist, dtype=np.int64).reshape(-1)
    if ell == width:
        return h.copy()
    return h.reshape(1 << ell, 1 << (width - ell)).sum(axis=1)


def zeros_from_hist(hist: np.ndarray, width: int) -> list[int]:
    """Z[l] = sum of even (l+1)-prefix counts (construct.py:238-239, structures.py:28-35)."""
    return [int(fold_to(hist, width, ell + 1)[0::2].sum()) for ell in range(width)]


def level_plan(hists: np.ndarray, kind: str, width: int, ell: int):
    """Merge plan of level ell (construct._merge_plan, construct.py:516-543).

    hists: (R, 2^width) per-rank histograms.  Returns pieces in destination
    order: (rank, local_start, length, global_start), empty pieces dropped.
    """
    hists = np.asarray(hists, dtype=np.int64)
    R = hists.shape[0]
    if ell == 0:
        lens = hists.reshape(R, -1).sum(axis=1)
        ranks = np.arange(R, dtype=np.int64)
        local = np.zeros(R, dtype=np.int64)
    else:
        counts = hists.reshape(R, 1 << ell, -1).sum(axis=2)  # (R, 2^ell), numeric prefix (fold_to per rank)
        order = bit_reversal_permutation(ell) if (kind == "wm" and ell >= 2) else np.arange(1 << ell)
        ordered = counts[:, order]
        local_starts = np.cumsum(ordered, axis=1) - ordered  # (R, groups) in interval order
        lens = ordered.T.reshape(-1)                          # group-major, rank-minor
        ranks = np.tile(np.arange(R, dtype=np.int64), 1 << ell)
        local = local_starts.T.reshape(-1)
    keep = lens > 0
    lens, ranks, local = lens[keep], ranks[keep], local[keep]
    gstart = np.cumsum(lens) - lens
    return ranks, local, lens, gstart


def exchange_plan(hists: np.ndarray, kind: str, width: int, n: int, local_ns, world: int):
    """Per level: which local bit range every source rank sends to every owner,
    and the owner's merge tasks.  Identical on every rank."""
    total_words = (n + 63) >> 6
    ranges = word_ranges(total_words, world)
    levels = []
    for ell in range(width):
        ranks, local, lens, gstart = level_plan(hists, kind, width, ell)
        per_dest = []
        for d, (w0, w1) in enumerate(ranges):
            b0, b1 = 64 * w0, min(64 * w1, n)
            if b1 <= b0:
                per_dest.append(None)
                continue
            # pieces intersecting [b0, b1)
            k0 = int(np.searchsorted(gstart + lens, b0, side="right"))
            k1 = int(np.searchsorted(gstart, b1, side="left"))
            sel = slice(k0, k1)
            pr, pl, pn, pg = ranks[sel], local[sel], lens[sel], gstart[sel]
            # local bit range needed from each source rank (contiguous: the local
            # level is the concatenation of the rank's pieces in interval order)
            lo = np.maximum(pl + np.maximum(b0 - pg, 0), 0)
            hi = pl + np.minimum(pg + pn, b1) - pg
            src_rng = []
            for r in range(world):
                m = pr == r
                if m.any():
                    src_rng.append((int(lo[m].min()) >> 6, (int(hi[m].max()) + 63) >> 6))
                else:
                    src_rng.append((0, 0))
            per_dest.append(dict(words=(w0, w1), ranks=pr, local=pl, lens=pn, gstart=pg, src=src_rng))
        levels.append(per_dest)
    return ranges, levels


def peer_plan_arrays(plans, owner: int, width: int):
    """This owner's merge tasks of every level, flattened for wvlt_merge_levels_peer:
    (bounds, bounds_off, starts, ranks, task_off).  Level l's tasks are
    [task_off[l], task_off[l+1]); its bounds (one more entry than tasks) start at
    bounds_off[l]; task t takes source rank ranks[t]'s local level l from bit
    starts[t]."""
    bounds, starts, ranks = [], [], []
    bounds_off, task_off = [], [0]
    boff = 0
    for ell in range(width):
        pd = plans[ell][owner]
        bounds_off.append(boff)
        if pd is None or len(pd["lens"]) == 0:
            task_off.append(task_off[-1])
            continue
        g, ln = np.asarray(pd["gstart"], dtype=np.int64), np.asarray(pd["lens"], dtype=np.int64)
        b = np.concatenate([g, [g[-1] + ln[-1]]])
        bounds.append(b)
        starts.append(np.asarray(pd["local"], dtype=np.int64))
        ranks.append(np.asarray(pd["ranks"], dtype=np.int32))
        boff += b.size
        task_off.append(task_off[-1] + ln.size)
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(1, dtype=dt)  # noqa: E731
    return (cat(bounds, np.int64), np.asarray(bounds_off, dtype=np.int64), cat(starts, np.int64),
            cat(ranks, np.int32), np.asarray(task_off, dtype=np.int64))


def owner_plan_arrays(hists: np.ndarray, kind: str, width: int, n: int, owner: int, world: int):
    """peer_plan_arrays(exchange_plan(...)[1], owner, width) computed for this owner
    alone (the p2p merge needs no per-source send ranges): per level the merge plan
    (level_plan) cut to the pieces that intersect the owner's bit range."""
    total_words = (n + 63) >> 6
    w0, w1 = word_ranges(total_words, world)[owner]
    b0, b1 = 64 * w0, min(64 * w1, n)
    bounds, starts, ranks = [], [], []
    bounds_off, task_off = [], [0]
    boff = 0
    for ell in range(width):
        bounds_off.append(boff)
        if b1 <= b0:
            task_off.append(task_off[-1])
            continue
        pr, pl, pn, pg = level_plan(hists, kind, width, ell)
        k0 = int(np.searchsorted(pg + pn, b0, side="right"))
        k1 = int(np.searchsorted(pg, b1, side="left"))
        if k1 <= k0:
            task_off.append(task_off[-1])
            continue
        g, ln = pg[k0:k1], pn[k0:k1]
        b = np.concatenate([g, [g[-1] + ln[-1]]])
        bounds.append(b)
        starts.append(pl[k0:k1])
        ranks.append(pr[k0:k1].astype(np.int32))
        boff += b.size
        task_off.append(task_off[-1] + (k1 - k0))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(1, dtype=dt)  # noqa: E731
    return (cat(bounds, np.int64), np.asarray(bounds_off, dtype=np.int64), cat(starts, np.int64),
            cat(ranks, np.int32), np.asarray(task_off, dtype=np.int64))


def merge_peer_host(arrays, sources, word_lo: int, word_hi: int, n: int, width: int):
    """Host restatement of wvlt_merge_levels_peer (test checker): ``sources[r][l]``
    is rank r's local level l (uint64 words).  Returns uint64 [width, word_hi - word_lo]."""
    bounds, boff, starts, ranks, toff = arrays
    out = np.zeros((width, max(word_hi - word_lo, 0)), dtype=np.uint64)
    for ell in range(width):
        t0, t1 = int(toff[ell]), int(toff[ell + 1])
        b = bounds[int(boff[ell]): int(boff[ell]) + (t1 - t0) + 1]
        for t in range(t1 - t0):
            lo, hi = max(int(b[t]), 64 * word_lo), min(int(b[t + 1]), 64 * word_hi, n)
            src = sources[int(ranks[t0 + t])][ell]
            for g in range(lo, hi):  # bit by bit: small test sizes only
                sp = int(starts[t0 + t]) + (g - int(b[t]))
                if (int(src[sp >> 6]) >> (sp & 63)) & 1:
                    out[ell, (g >> 6) - word_lo] |= np.uint64(1) << np.uint64(g & 63)
    return out


def plan_from_borders_host(rows_borders, local_ns, kind: str, width: int):
    """Host restatement of the device plan (wvlt_peer_plan, test checker): every
    level's (group in interval order, rank) pieces from the ranks' node borders.
    rows_borders[r] is rank r's borders array (wvlt_build_device layout).
    Returns (bounds, bounds_off, starts, ranks, task_off) like owner_plan_arrays,
    but uncut and with empty pieces kept."""
    R = len(local_ns)
    bounds, starts, ranks = [], [], []
    for ell in range(width):
        ng = 1 << ell
        if ell == 0:
            st = np.zeros((1, R), dtype=np.int64)
            ln = np.asarray(local_ns, dtype=np.int64).reshape(1, R)
        else:
            order = bit_reversal_permutation(ell) if (kind == "wm" and ell >= 2) else np.arange(ng)
            blk = np.stack([np.asarray(rows_borders[r], dtype=np.int64)[(1 << ell) - 2: (1 << (ell + 1)) - 2]
                            for r in range(R)], axis=1)  # [prefix, rank]
            st = blk[order]                                # [interval order, rank]
            nxt = np.vstack([st[1:], np.asarray(local_ns, dtype=np.int64).reshape(1, R)])
            ln = nxt - st
        g = st.sum(axis=1, keepdims=True)
        within = np.cumsum(ln, axis=1) - ln
        b = (g + within).reshape(-1)
        bounds.append(np.concatenate([b, [int(np.sum(local_ns))]]))
        starts.append(st.reshape(-1))
        ranks.append(np.tile(np.arange(R, dtype=np.int32), ng))
    task_off = np.array([R * ((1 << ell) - 1) for ell in range(width + 1)], dtype=np.int64)
    bounds_off = np.array([R * ((1 << ell) - 1) + ell for ell in range(width)], dtype=np.int64)
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(1, dtype=dt)  # noqa: E731
    return cat(bounds, np.int64), bounds_off, cat(starts, np.int64), cat(ranks, np.int32), task_off


def build_sharded(local_text, sigma: int, kind: str = "wm", group=None, *, ops=None, gather: bool = False,
                  transport: str = "nccl", comm_device=None):
    """Sharded build over the ranks of ``group`` (default: the world group).

    Every rank passes its own contiguous shard of the text (rank order = text
    order).  Returns this rank's ShardedResult; with ``gather`` rank 0 also gets
    the full level words (attribute ``full_words``).  ``ops`` supplies the local
    build and the merge; the default uses this rank's CUDA device.

    ``transport``: "nccl" moves the needed bit segments with one all_to_all and
    shift-merges them (wvlt_merge_bits); "p2p" builds every rank's local levels in
    peer-mapped memory and lets each owner assemble its words straight from the
    peers' levels in one kernel (wvlt_merge_levels_peer) -- the exchange fused
    into the merge, no staging copy.  The p2p merge plan is computed on the
    device from the all-gathered node borders (wvlt_peer_plan): no host planning.

    ``comm_device``: where the collectives' tensors live (default: the build
    device).  "cpu" stages them through host memory, for a gloo group (the
    one-GPU multi-process tests); the builds and merges stay on the GPU.
    """
    import torch
    import torch.distributed as dist

    if kind not in ("wt", "wm"):
        raise ValueError(f"unknown structure kind {kind!r}")
    sigma = int(sigma)
    if sigma < 1:
        raise ValueError("alphabet size must be at least 1")
    ops = ops or CudaOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = ops.device
    cdev = torch.device(comm_device) if comm_device is not None else dev
    width = code_width(sigma)

    n_local = int(local_text.numel() if hasattr(local_text, "numel") else np.asarray(local_text).size)
    ns = torch.zeros(world, dtype=torch.int64, device=cdev)
    mine = torch.tensor([n_local], dtype=torch.int64, device=cdev)
    dist.all_gather_into_tensor(ns, mine, group=group)
    local_ns = [int(v) for v in ns.cpu().tolist()]
    n = sum(local_ns)

    if transport not in ("nccl", "p2p"):
        raise ValueError(f"unknown transport {transport!r}")
    total_words = (n + 63) >> 6
    ranges = word_ranges(total_words, world)
    w0, w1 = ranges[rank]
    if transport == "p2p" and width > 0:
        return _build_sharded_p2p(local_text, sigma, kind, group, ops, gather, local_ns, ns, n, rank, world, ranges,
                                  cdev)

    # 1. local build (no communication)
    words, hist, bad = ops.local_build(local_text, sigma, kind)
    # 2. histograms (+ each rank's range flag) -> plan: one all_gather, one host read
    if torch.is_tensor(bad):
        flag = (bad.reshape(-1)[:1].to(device=cdev, dtype=torch.int64) & 1)
    else:
        flag = torch.tensor([1 if bad else 0], dtype=torch.int64, device=cdev)
    mine_h = torch.cat([hist.reshape(-1).to(device=cdev, dtype=torch.int64), flag])
    allh = torch.empty((world, (1 << width) + 1), dtype=torch.int64, device=cdev)
    dist.all_gather_into_tensor(allh, mine_h.reshape(1, -1), group=group)
    gathered = allh.cpu().numpy()
    if gathered[:, -1].any():
        raise ValueError(f"symbols must lie in [0, {sigma})")
    hists = np.ascontiguousarray(gathered[:, :-1])
    ghist = hists.sum(axis=0)
    zeros = zeros_from_hist(ghist, width) if width else []
    # the merge kernels write every owned word (padding bits included)
    owned = torch.empty((width, max(w1 - w0, 0)), dtype=torch.int64, device=dev)
    if width == 0 or n == 0:
        return ShardedResult(n, sigma, kind, width, w0, w1, owned, zeros, ghist)

    plans = exchange_plan(hists, kind, width, n, local_ns, world)[1]
    # 3. one all_to_all for every level: the send buffer is grouped by
    #    destination (levels in order inside), so the receive buffer is grouped
    #    by source rank with levels in order inside
    send_parts, send_sizes = [], [0] * world
    recv_sizes = [0] * world
    for d in range(world):
        for ell in range(width):
            pd = plans[ell][d]
            if pd is None:
                continue
            a, b = pd["src"][rank]
            if b > a:
                send_parts.append(words[ell, a:b])
                send_sizes[d] += b - a
    for ell in range(width):
        pd = plans[ell][rank]
        if pd is not None:
            for r in range(world):
                a, b = pd["src"][r]
                recv_sizes[r] += max(b - a, 0)
    send = torch.cat(send_parts).to(cdev) if send_parts else torch.zeros(0, dtype=torch.int64, device=cdev)
    recv = torch.empty(sum(recv_sizes), dtype=torch.int64, device=cdev)
    dist.all_to_all_single(recv, send, recv_sizes, send_sizes, group=group)
    recv = recv.to(dev)

    # receive-buffer offsets: segments arrive grouped by source rank, level-major inside
    seg_base = np.cumsum([0] + recv_sizes[:-1])
    cursor = list(seg_base)
    # 4. shift-merge every owned level range
    for ell in range(width):
        pd = plans[ell][rank]
        if pd is None:
            continue
        off = np.zeros(world, dtype=np.int64)  # word offset of (ell, r) segment in recv
        for r in range(world):
            a, b = pd["src"][r]
            off[r] = cursor[r] - a  # so that local word x of rank r is recv[off[r] + x]
            cursor[r] += max(b - a, 0)
        pr = pd["ranks"]
        src_starts = 64 * off[pr] + pd["local"]
        bounds = np.concatenate([pd["gstart"], [pd["gstart"][-1] + pd["lens"][-1]]]).astype(np.int64)
        ops.merge(owned[ell], w0, w1, n, bounds, src_starts.astype(np.int64), recv)
    res = ShardedResult(n, sigma, kind, width, w0, w1, owned, zeros, ghist)
    if gather:
        res.full_words = _gather_levels(owned, ranges, width, total_words, rank, world, group, dev, cdev)
    return res


def _build_sharded_p2p(local_text, sigma, kind, group, ops, gather, local_ns, ns, n, rank, world, ranges, cdev):
    """p2p transport: local levels in peer-mapped memory, plan and merge on the device."""
    import torch
    import torch.distributed as dist

    dev = ops.device
    width = code_width(sigma)
    nb = 1 << width
    w0, w1 = ranges[rank]
    total_words = (n + 63) >> 6
    lnws = [(v + 63) >> 6 for v in local_ns]
    # 1. local build straight into this rank's peer-visible buffer, with its
    #    histogram, node borders (= the rank's local group starts) and zero counts
    hdl_ptrs, buf = ops.peer_buffer(width * max(lnws), group, cdev)
    lb = ops.local_build(local_text, sigma, kind, out_words=buf[: width * lnws[rank]], borders=True)
    words, hist, bad, borders, zeros_local = lb
    # 2. one all_gather of [histogram | borders | zero counts | range flag] per rank
    flag = (bad.reshape(-1)[:1].to(torch.int64) & 1) if torch.is_tensor(bad) else         torch.tensor([1 if bad else 0], dtype=torch.int64, device=dev)
    nbd = max(nb - 2, 0)
    row = torch.cat([hist.reshape(-1).to(torch.int64), borders.reshape(-1)[:nbd].to(torch.int64),
                     zeros_local.reshape(-1)[:width].to(torch.int64), flag.reshape(-1)]).to(cdev)
    rowlen = row.numel()
    allrows = torch.empty((world, rowlen), dtype=torch.int64, device=cdev)
    dist.all_gather_into_tensor(allrows, row.reshape(1, -1), group=group)
    tail = allrows[:, nb + nbd:].cpu().numpy()  # per rank: zero counts + flag (one small host read)
    if tail[:, -1].any():
        raise ValueError(f"symbols must lie in [0, {sigma})")
    zeros = [int(z) for z in tail[:, :width].sum(axis=0)]  # zero counts add over shards
    rows_dev = allrows.to(dev)
    ghist = rows_dev[:, :nb].sum(dim=0)
    owned = torch.empty((width, max(w1 - w0, 0)), dtype=torch.int64, device=dev)
    if n > 0:
        # 3. the merge plan of every level on the device (wvlt_peer_plan), then
        # 4. one kernel per owner reads the peers' local levels directly.  The
        #    all_gather above is ordered after every rank's local build, so the
        #    peers' levels are complete once it has finished here.
        plan = ops.device_plan(rows_dev, rowlen, nb, ns.to(dev), world, width, kind)
        level_src = ops.level_sources(hdl_ptrs, lnws, width, world)
        ops.merge_peer_device(owned, w0, w1, n, plan, level_src, world)
    # peers may reuse their buffers only after every owner has read them (a
    # host-staged completion collective is not ordered after the merge kernel)
    if cdev.type != "cuda":
        torch.cuda.current_stream(dev).synchronize()
    done = torch.zeros(1, dtype=torch.int64, device=cdev)
    dist.all_reduce(done, group=group)
    res = ShardedResult(n, sigma, kind, width, w0, w1, owned, zeros, ghist)
    if gather:
        res.full_words = _gather_levels(owned, ranges, width, total_words, rank, world, group, dev, cdev)
    return res


def _gather_levels(owned, ranges, width, total_words, rank, world, group, dev, cdev=None):
    """Assemble the full levels on rank 0 (owned ranges padded to equal size for gather)."""
    import torch
    import torch.distributed as dist

    cdev = cdev if cdev is not None else dev
    sizes = [(b - a) * width for a, b in ranges]
    mx = max(sizes) if sizes else 0
    flat = torch.zeros(mx, dtype=torch.int64, device=cdev)
    flat[: sizes[rank]] = owned.reshape(-1).to(cdev)
    if rank == 0:
        parts = [torch.empty(mx, dtype=torch.int64, device=cdev) for _ in range(world)]
        dist.gather(flat, parts, dst=0, group=group)
        full = torch.empty((width, total_words), dtype=torch.int64, device=dev)
        for (a, b), p, sz in zip(ranges, parts, sizes):
            full[:, a:b] = p[:sz].reshape(width, b - a).to(dev)
        return full
    dist.gather(flat, None, dst=0, group=group)
    return None


class CudaOps:
    """Local build + merge on this rank's CUDA device (hand-written kernels).

    ``peer``: how the p2p transport maps every rank's local levels into every
    peer -- "symm" (torch symmetric memory over NVLink, the NCCL product path)
    or "ipc" (CUDA IPC handles exchanged through the process group; several
    processes sharing one GPU in the one-GPU multi-rank tests)."""

    def __init__(self, device=None, peer: str = "symm"):
        import torch

        from .device import DeviceBuilder

        if peer not in ("symm", "ipc"):
            raise ValueError(f"unknown peer mapping {peer!r}")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.builder = DeviceBuilder(self.device)
        self.peer = peer
        self._peer = None   # (peer pointers, buffer[, keep-alive]) of the p2p transport, reused while large enough
        self._plan = None   # device plan buffers, reused while the shape matches
        self._src = None    # ((pointers, lnws, width), device level-source table)

    def peer_buffer(self, words: int, group=None, comm_device=None):
        """An int64 buffer of at least ``words`` on every rank of ``group``, mapped
        into every peer (collective when it has to grow: every rank asks for the
        same size).  Returns (per-rank base pointers, this rank's buffer)."""
        import torch
        import torch.distributed as dist

        if self._peer is None or self._peer[1].numel() < words:
            self._peer = None
            self._src = None
            if self.peer == "symm":
                from torch.distributed import _symmetric_memory as symm_mem

                buf = symm_mem.empty(max(int(words), 1), dtype=torch.int64, device=self.device)
                hdl = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
                self._peer = ([int(p) for p in hdl.buffer_ptrs], buf, hdl)
            else:
                from torch.multiprocessing.reductions import reduce_tensor

                buf = torch.empty(max(int(words), 1), dtype=torch.int64, device=self.device)
                world, rank = dist.get_world_size(group), dist.get_rank(group)
                handles = [None] * world
                dist.all_gather_object(handles, reduce_tensor(buf), group=group)
                peers = [buf if r == rank else fn(*args) for r, (fn, args) in enumerate(handles)]
                self._peer = ([int(t.data_ptr()) for t in peers], buf, peers)
        return self._peer[0], self._peer[1]

    def local_build(self, text, sigma: int, kind: str, out_words=None, borders: bool = False):
        import torch

        if not isinstance(text, torch.Tensor):
            from .construct import _device_text

            text = torch.from_numpy(_device_text(np.ascontiguousarray(np.asarray(text)), sigma))
        text = text.to(self.device)
        outputs = None
        if out_words is not None or borders:  # levels into a caller buffer (peer-mapped for the p2p merge)
            lw, zeros, hist, bd, status = self.builder.alloc_outputs(int(text.numel()), sigma, borders=borders)
            if out_words is not None:
                lw = out_words.view(lw.shape)
            if borders and bd is None:
                bd = torch.zeros(1, dtype=torch.int64, device=self.device)
            outputs = (lw, zeros, hist, bd, status)
        res = self.builder.build(text, sigma, kind, histogram=True, borders=borders, check=False, outputs=outputs)
        # the range status stays on the device (read with the histograms, no extra sync)
        bad = res.status if res.status is not None else False
        if borders:
            return res.level_words, res.hist, bad, res.borders, res.zeros
        return res.level_words, res.hist, bad

    def merge(self, dst_row, word_lo: int, word_hi: int, n_bits: int, bounds, src_starts, src):
        import torch

        b = torch.from_numpy(bounds).to(self.device)
        s = torch.from_numpy(src_starts).to(self.device)
        self.builder.merge_bits(dst_row, word_lo, word_hi, n_bits, b, s, src, dst_offset_words=word_lo)

    def device_plan(self, rows, row_stride: int, borders_col: int, ns_dev, nranks: int, width: int, kind: str):
        """wvlt_peer_plan into cached device buffers: (bounds, bounds_off, starts, ranks, task_off).
        ``ns_dev``: int64 device tensor of the ranks' symbol counts."""
        import torch

        from . import _lib

        ntask = nranks * ((1 << width) - 1)
        key = (nranks, width)
        if self._plan is None or self._plan[0] != key:
            dev = self.device
            self._plan = (key, (torch.empty(ntask + width, dtype=torch.int64, device=dev),
                                torch.empty(max(width, 1), dtype=torch.int64, device=dev),
                                torch.empty(max(ntask, 1), dtype=torch.int64, device=dev),
                                torch.empty(max(ntask, 1), dtype=torch.int32, device=dev),
                                torch.empty(width + 1, dtype=torch.int64, device=dev)))
        bounds, boff, starts, ranks, toff = self._plan[1]
        ns_dev = ns_dev.to(device=self.device, dtype=torch.int64).contiguous()
        rc = _lib.load().wvlt_peer_plan(rows.data_ptr(), int(row_stride), int(borders_col), ns_dev.data_ptr(),
                                        int(nranks), int(width), _lib.KINDS[kind], bounds.data_ptr(),
                                        starts.data_ptr(), ranks.data_ptr(), boff.data_ptr(), toff.data_ptr(),
                                        torch.cuda.current_stream(self.device).cuda_stream)
        _lib.check(rc)
        return bounds, boff, starts, ranks, toff

    def level_sources(self, ptrs, lnws, width: int, nranks: int):
        """Device table of every (level, rank)'s local level address, cached per buffer layout."""
        import torch

        key = (tuple(ptrs), tuple(lnws), width)
        if self._src is None or self._src[0] != key:
            tab = np.array([[ptrs[r] + 8 * ell * lnws[r] for r in range(nranks)] for ell in range(width)],
                           dtype=np.int64)
            self._src = (key, torch.from_numpy(tab.reshape(-1)).to(self.device))
        return self._src[1]

    def merge_peer_device(self, owned, word_lo: int, word_hi: int, n_bits: int, plan, level_src, nranks: int):
        """wvlt_merge_levels_peer with a device plan and a device level-source table."""
        import torch

        from . import _lib

        bounds, boff, starts, ranks, toff = plan
        width = int(owned.shape[0])
        rc = _lib.load().wvlt_merge_levels_peer(
            owned.data_ptr(), int(owned.shape[1]) if owned.dim() == 2 else 0, width, int(word_lo), int(word_hi),
            int(n_bits), bounds.data_ptr(), boff.data_ptr(), starts.data_ptr(), ranks.data_ptr(), toff.data_ptr(),
            level_src.data_ptr(), int(nranks), torch.cuda.current_stream(self.device).cuda_stream)
        _lib.check(rc)

    def merge_peer(self, owned, word_lo: int, word_hi: int, n_bits: int, arrays, level_src, nranks: int):
        """wvlt_merge_levels_peer into ``owned`` [width, word_hi - word_lo] from host plan
        arrays (owner_plan_arrays); ``level_src`` int64 [width, nranks] device addresses
        of every rank's local levels."""
        import torch

        dev = self.device
        bounds, boff, starts, ranks, toff = arrays
        plan = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (bounds, boff, starts, ranks, toff))
        src = torch.from_numpy(np.ascontiguousarray(level_src, dtype=np.int64).reshape(-1)).to(dev)
        self.merge_peer_device(owned, word_lo, word_hi, n_bits, plan, src, nranks)
