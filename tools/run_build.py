"""Run a few device builds of one config (for ncu / compute-sanitizer captures).

    python tools/run_build.py --config c2 --log2n 26 --kind wm --iters 2
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--log2n", type=int, default=None)
    ap.add_argument("--kind", default=None)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--variant", default=None, help="a tools/variants/<name>.so tuning build instead of the product library")
    a = ap.parse_args()
    if a.variant:
        from paper_1702_07578_b200 import _lib

        _lib.load_variant(ROOT / "tools" / "variants" / f"{a.variant}.so")
    from paper_1702_07578_b200.device import DeviceBuilder

    cfg = workloads.CONFIGS[a.config]
    n = (1 << a.log2n) if a.log2n else cfg["n"]
    text = workloads.generate(a.config, n=n)
    b = DeviceBuilder()
    outs = b.alloc_outputs(n, cfg["sigma"])
    kind = a.kind or cfg["kind"]
    for _ in range(a.iters):
        b.build(text, cfg["sigma"], kind, outputs=outs, check=True)
    torch.cuda.synchronize()
    print("ok", a.config, n, kind)


if __name__ == "__main__":
    main()
