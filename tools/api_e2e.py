"""Time the reference-facing Python API (construct.build_structure) on a host
numpy text: pageable input as a caller passes it, output words into numpy."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1702_07578_b200 import construct  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = workloads.CONFIGS[cfg]
text = workloads.generate(cfg).cpu().numpy()
for kind in ("wm", "wt"):
    construct.build_structure(text[: 1 << 20], c["sigma"], kind)  # warm-up
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        st = construct.build_structure(text, c["sigma"], kind)
        ts.append(time.perf_counter() - t0)
    print(cfg, kind, "build_structure ms", [round(t * 1e3, 1) for t in ts], "n", text.size)
