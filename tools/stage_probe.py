"""wvlt_build_host with pinned / pageable text and output words (c2 shape)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402

if len(sys.argv) > 1:  # a tools/variants/<name>.so tuning build
    from paper_1702_07578_b200 import _lib

    _lib.load_variant(Path(__file__).resolve().parents[1] / "tools" / "variants" / f"{sys.argv[1]}.so")
    print("variant", sys.argv[1])
from paper_1702_07578_b200.device import DeviceBuilder  # noqa: E402

text_d = workloads.generate("c2")
n = text_d.numel()
pinned_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pinned_in.copy_(text_d)
pageable_in = text_d.cpu().numpy().copy()
pin_out = torch.empty((8, n // 64), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
touched_out = np.ones((8, n // 64), dtype=np.uint64)
b = DeviceBuilder()


def run(tin, out_fn, k=3):
    b.build_host(tin, 256, "wm", out_words=out_fn())
    ts = []
    for _ in range(k):
        o = out_fn()
        t0 = time.perf_counter()
        b.build_host(tin, 256, "wm", out_words=o)
        ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    return ts


pin_in_np = pinned_in.numpy()
print("pinned in, pinned out", run(pin_in_np, lambda: pin_out))
print("pageable in, pinned out", run(pageable_in, lambda: pin_out))
print("pinned in, pageable touched out", run(pin_in_np, lambda: touched_out))
print("pinned in, pageable fresh out", run(pin_in_np, lambda: np.empty((8, n // 64), dtype=np.uint64)))
print("pageable in, pageable fresh out", run(pageable_in, lambda: np.empty((8, n // 64), dtype=np.uint64)))
