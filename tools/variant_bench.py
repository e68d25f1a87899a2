"""Benchmark tuning variants without touching the product library.

    python tools/variant_bench.py --build name:DEF=1,DEF2=3 ...   (here, nvcc only)
    python tools/variant_bench.py --run name ... [--config c2]      (GPU box)

Variants are built by ``_build.build_variant`` into tools/variants/<name>.so
(git-ignored) and bound with ``_lib.load_variant`` in a child process each;
the product ``_wvlt_b200.so`` is never overwritten.  "base" runs the product
library.
"""

from __future__ import annotations

import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def child(name: str, config: str, steps: int) -> None:
    from paper_1702_07578_b200 import _lib

    if name != "base":
        _lib.load_variant(ROOT / "tools" / "variants" / f"{name}.so")
    import torch

    import workloads
    from paper_1702_07578_b200.device import DeviceBuilder

    cfg = workloads.CONFIGS[config]
    text = workloads.generate(config)
    b = DeviceBuilder()
    outs = b.alloc_outputs(cfg["n"], cfg["sigma"])
    for _ in range(3):
        b.build(text, cfg["sigma"], cfg["kind"], outputs=outs, check=False)
    _lib.profile_enable(True)
    stages = {}
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        b.build(text, cfg["sigma"], cfg["kind"], outputs=outs, check=False)
    e1.record(s)
    torch.cuda.synchronize()
    for k, v in _lib.profile_read():
        stages[k] = round(v, 4)
    lw = outs[0]
    w = torch.arange(1, lw.numel() + 1, device=lw.device, dtype=torch.int64)
    digest = [int((lw.reshape(-1) * w).sum()), int(lw.reshape(-1).sum()), int(outs[1].sum())]
    print(json.dumps({"variant": name, "config": config, "ms": e0.elapsed_time(e1) / steps, "stages_ms": stages,
                      "digest": digest}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", nargs="*", default=[])
    ap.add_argument("--run", nargs="*", default=[])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--child", default=None)
    a = ap.parse_args()
    if a.child:
        child(a.child, a.config, a.steps)
        return
    from paper_1702_07578_b200 import _build

    for spec in a.build:
        name, _, defs = spec.partition(":")
        print(_build.build_variant(name, [d for d in defs.split(",") if d]))
    for name in a.run:
        subprocess.run([sys.executable, __file__, "--child", name, "--config", a.config, "--steps", str(a.steps)])


if __name__ == "__main__":
    main()
