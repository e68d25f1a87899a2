"""Pageable host <-> device copy rates (1 GiB), fresh vs touched host memory, and host memcpy rate."""
import time

import numpy as np
import torch

n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
src = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)


def t(f, k=3):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return [round(x, 1) for x in ts]


print("h2d pageable ms", t(lambda: d.copy_(torch.from_numpy(src))))
touched = np.ones(n, dtype=np.uint8)
print("d2h pageable touched ms", t(lambda: torch.from_numpy(touched).copy_(d)))


def fresh():
    out = np.empty(n, dtype=np.uint8)
    torch.from_numpy(out).copy_(d)


print("d2h pageable fresh ms", t(fresh))
print("np.empty + touch ms", t(lambda: np.empty(n, dtype=np.uint8).fill(0)))
dst = np.empty_like(src)
print("host memcpy 1 thread ms", t(lambda: np.copyto(dst, src)))
import os
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
