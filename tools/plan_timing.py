"""Time the sharded build's merge plan: device (wvlt_peer_plan) vs the host numpy
restatement (owner_plan_arrays), at w = 20 with R = 8 ranks (c5 sharded 8 ways)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import oracle
from paper_1702_07578_b200.distributed import CudaOps, owner_plan_arrays

w, R = 20, 8
rng = np.random.default_rng(1)
hists = rng.integers(0, 300, (R, 1 << w)).astype(np.int64)
rows = np.stack([np.concatenate([h, oracle.borders(h, w, "wm")]) for h in hists])
ns = torch.tensor(hists.sum(1), device="cuda")
rows_d = torch.from_numpy(rows).cuda()
ops = CudaOps()
for _ in range(3):
    ops.device_plan(rows_d, rows.shape[1], 1 << w, ns, R, w, "wm")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ops.device_plan(rows_d, rows.shape[1], 1 << w, ns, R, w, "wm")
e1.record()
torch.cuda.synchronize()
dev_ms = e0.elapsed_time(e1) / 10
t0 = time.perf_counter()
owner_plan_arrays(hists, "wm", w, int(hists.sum()), 0, R)
host_ms = (time.perf_counter() - t0) * 1e3
print(json.dumps({"w": w, "ranks": R, "device_plan_ms": dev_ms, "host_owner_plan_ms": host_ms,
                  "host_work_per_build_ms": 0.0,
                  "note": "device plan: one wvlt_peer_plan launch for every level; no host planning, no plan upload"}))
