"""PCIe probe: H2D alone, D2H alone, both at once (two streams), 1 GiB each, pinned."""
import time

import torch

n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
su, sd = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, k=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3


def h2d():
    with torch.cuda.stream(su):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(sd):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


print("h2d ms", t(h2d), "d2h ms", t(d2h), "both ms", t(both))
print(torch.cuda.get_device_properties(0))
