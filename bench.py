"""Benchmark: WT/WM construction throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One step = one full wavelet-matrix build of configs[1] (c2: n=2^30 uint8,
sigma=256, Zipf(1.1)) with the text already resident in HBM: histogram (K1),
tables (K2) and the fused level passes (K3), output level words + zero counts.
Prints one JSON line (rank 0).

``value``     whole-job symbols/s of the device-resident build, CUDA events on
              the launch stream, max over ranks.
``e2e``       the same metric through the reference-facing C ABI with pinned HOST
              buffers: K builds queued through wvlt_build_host_batch (upload of
              text i+1 / build i / download of build i-1 overlapped), every
              build's H2D of the text and D2H of all level words + zeros inside
              the timed region; ``latency_ms`` = one wvlt_build_host call.
``roofline``  the dominant kernel (longest stage, from per-stage CUDA events):
              algorithmic bytes / its average duration vs MEASURED_PEAKS.json.
``cpu_baseline`` the oracle's port of the reference ps builder
              (construct.py:322-387) on all host cores over a bounded sample.
``--impl reference`` times that CPU path alone (rank 0; other ranks exit 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "WT+WM build input symbols/sec (n=2^30, σ=256) and % of HBM bytes-moved roofline"
UNIT = "symbols/s"
KMAX = 4


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def code_width(sigma: int) -> int:
    return max(sigma - 1, 0).bit_length()


def pass_plan(n: int, sym_bytes: int, sigma: int, kind: str):
    """Mirror of the device plan (make_plan() / k8_eligible() in csrc): (level, K, in_bytes, out_bytes) per pass.
    The fused stages (k8 / k16 / k32) get their first level from their counting kernel (hist8/16/32)."""
    w = code_width(sigma)
    if sym_bytes == 1 and 2 <= w <= 8 and 0 < n < (1 << 32) - 64:
        return [(0, w, 1, 0)]  # k8.cuh: every level in one fused pass
    vbits = 8 * sym_bytes
    bb = lambda b: 1 if b <= 8 else 2 if b <= 16 else 4  # noqa: E731
    out, ell = [], 0
    fused = kind == "wm" and w > 8 and 0 < n < (1 << 32) - 64  # make_plan(): fused 4-/2-byte passes + byte tail
    cur = bb(w) if 8 * sym_bytes < w else sym_bytes  # element bytes of the next stage's input (widened text)
    while ell < w:
        live = w - ell
        if fused and live <= 8:
            out.append((ell, live, 1, 0))
            break
        if fused and 18 <= live <= 24 and cur == 4:  # k32.cuh: fused 4-byte pass, 2-byte output
            out.append((ell, live - 16, 4, 2))
            ell, cur = w - 16, 2
            continue
        if fused and 10 <= live <= 16 and cur == 2:  # k16.cuh: fused 2-byte pass, byte output
            out.append((ell, live - 8, 2, 1))
            ell, cur = w - 8, 1
            continue
        K = min(KMAX, live)
        live_in = live if kind == "wm" else w
        live_out = (live - K) if kind == "wm" else w
        ib = sym_bytes if ell == 0 else bb(min(live_in, vbits))
        ob = bb(min(live_out, vbits)) if ell + K < w else 0
        out.append((ell, K, ib, min(ob, ib)))
        cur = min(ob, ib)
        ell += K
    return out


def stage_bytes(name: str, n: int, sym_bytes: int, sigma: int, kind: str) -> float:
    """Algorithmic bytes a stage must move."""
    w = code_width(sigma)
    if name == "hist":
        return n * sym_bytes
    if name == "memset":
        return w * ((n + 63) // 64) * 8
    if name.startswith("pass"):
        ell, K, ib, ob = pass_plan(n, sym_bytes, sigma, kind)[int(name[4:])]
        return n * ib + n * ob + K * ((n + 63) // 64) * 8
    return 0.0


def fused_stage(plan_entry, n: int, sym_bytes: int, sigma: int, kind: str) -> bool:
    """True for the fused k8 / k16 / k32 stages (their first level comes from the stage's counting kernel)."""
    ell, K, ib, ob = plan_entry
    w = code_width(sigma)
    if sym_bytes == 1 and 2 <= w <= 8 and 0 < n < (1 << 32) - 64:
        return True
    fused = kind == "wm" and w > 8 and 0 < n < (1 << 32) - 64
    return fused and ((ob == 0 and ib == 1 and w - ell <= 8) or (ib, ob) in ((4, 2), (2, 1)))


def stage_levels(name: str, n: int, sym_bytes: int, sigma: int, kind: str) -> int:
    """Levels a stage's kernel emits (SURVEY 8d charges n s + n/8 bytes per level)."""
    plan = pass_plan(n, sym_bytes, sigma, kind)
    if name.startswith("pass"):
        e = plan[int(name[4:])]
        return e[1] - (1 if fused_stage(e, n, sym_bytes, sigma, kind) else 0)
    single = len(plan) == 1 and plan[0][2] == 1 and plan[0][3] == 0 and plan[0][0] == 0
    if name == "hist":  # the byte path's counting kernel (hist8) writes level 0
        return 1 if single and fused_stage(plan[0], n, sym_bytes, sigma, kind) else 0
    if name.startswith("scan") and name[4:].isdigit():  # wide fused stages: counting kernel + tables, first level
        p = int(name[4:])
        return 1 if not single and p < len(plan) and fused_stage(plan[p], n, sym_bytes, sigma, kind) else 0
    return 0


def metric_bytes(n: int, sym_bytes: int, sigma: int) -> float:
    """B = L (n s + 8 ceil(n/64)), text read once per level + level bits."""
    w = code_width(sigma)
    return w * (n * sym_bytes + 8 * ((n + 63) // 64))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[2:6]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    return "unknown"


REF_NOTE = ("the reference package (wvlt: Python + numba) cannot run on the GPU box: numba is not installed in "
            "this image and there is no network; its algorithms run as the oracle's C restatement (kind 'port'), "
            "pinned to the reference's own golden vectors (tests/test_oracle_golden.py)")


def cpu_baseline(text_host: np.ndarray, sigma: int, kind: str, sample: int, runs: int = 3, algo: str = "ps",
                 threads: int | None = None):
    """Oracle port of a reference builder (ps by default) on all host cores over text[:sample]."""
    import oracle

    threads = threads or cpu_threads()
    piece = np.ascontiguousarray(text_host[:sample])
    oracle.build(piece[: 1 << 16], sigma, kind, algo, threads)  # warm-up
    times = []
    for _ in range(runs):
        t0 = time.perf_counter()
        oracle.build(piece, sigma, kind, algo, threads)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    src = {"ps": "construct.py:322-387", "pc": "construct.py:292-319", "ddps": "construct.py:437-543",
           "ddpc": "construct.py:437-543"}[algo]
    return {"value": piece.size / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"{'all' if piece.size == text_host.size else 'first'} {piece.size} symbols of the same "
                       f"{kind.upper()} text, oracle {algo} (restatement of {src}) with {threads} POSIX "
                       f"thread{'s' if threads > 1 else ''}, median of {runs}"),
            "cpu_model": cpu_model(), "reference_package": REF_NOTE, "seconds_per_build": t}


def cpu_variants(text_host: np.ndarray, sigma: int, kind: str, pc_sample: int):
    """BASELINE.md §4's other CPU figures: ddps / ddpc at all host threads on the
    whole text, pc on one thread over a bounded sample (it is ~50x slower)."""
    out = {}
    for algo in ("ddps", "ddpc"):
        r = cpu_baseline(text_host, sigma, kind, text_host.size, runs=1, algo=algo)
        out[algo] = {"value": r["value"], "cores": r["cores"], "sample": r["sample"]}
    r = cpu_baseline(text_host, sigma, kind, min(pc_sample, text_host.size), runs=1, algo="pc", threads=1)
    out["pc_p1"] = {"value": r["value"], "cores": 1, "sample": r["sample"]}
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port, all host threads)."""
    import torch
    import workloads

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = workloads.CONFIGS[args.config]
    sample = min(cfg["n"], args.cpu_sample) if args.cpu_sample else cfg["n"]
    text = workloads.generate(args.config, device="cuda" if torch.cuda.is_available() else "cpu")
    host = text.cpu().numpy()
    del text
    kind = args.kind or cfg["kind"]
    for _ in range(args.warmup):
        cpu_baseline(host, cfg["sigma"], kind, min(sample, 1 << 20), runs=1)
    times = []
    for _ in range(args.steps):
        r = cpu_baseline(host, cfg["sigma"], kind, sample, runs=1)
        times.append(r["seconds_per_build"])
    t = sum(times) / len(times)
    value = sample / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8" if cfg["dtype"] == torch.uint8 else str(cfg["dtype"]),
        "data": "synthetic", "config": {"workload": args.config, "description": workloads.DESCRIPTIONS[args.config],
                                         "kind": kind, "n": sample, "sigma": cfg["sigma"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_threads(), "kind": "port",
                         "sample": (f"{'the whole' if sample == cfg['n'] else f'first {sample} symbols of the'} "
                                    f"{args.config} text per step (same config as the GPU arm); oracle ps = "
                                    "restatement of the reference ps builder (construct.py:322-387), all host threads"),
                         "cpu_model": cpu_model(), "reference_package": REF_NOTE},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "same_config": sample == cfg["n"],
    }
    if not args.no_variants:
        line["cpu_variants"] = cpu_variants(host, cfg["sigma"], kind, 1 << 26)
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--kind", default=None, choices=[None, "wt", "wm"])
    ap.add_argument("--cpu-sample", type=int, default=0, help="symbols of the CPU legs (0 = the whole config text)")
    ap.add_argument("--borders", action="store_true", help="also emit the node borders (always on for c1)")
    ap.add_argument("--no-variants", action="store_true", help="skip the ddps / ddpc / pc p=1 CPU figures")
    ap.add_argument("--no-api", action="store_true", help="skip the build_structure (numpy in, BitVectors out) figure")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-wt", action="store_true")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="N = 1 (default): time CUDA-graph replays of the captured build (DeviceBuilder.capture: "
                         "the build's launches recorded once, replayed with one launch)")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="N = 1: launch the build's kernels one by one")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: merge over peer memory (symmetric memory, one kernel) or NCCL all_to_all + merge")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import workloads
    from paper_1702_07578_b200 import _lib
    from paper_1702_07578_b200.device import DeviceBuilder

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg = workloads.CONFIGS[args.config]
    kind = args.kind or cfg["kind"]
    sigma, n = cfg["sigma"], cfg["n"]
    sym_bytes = torch.empty(0, dtype=cfg["dtype"]).element_size()
    # weak scaling: every rank builds its own n-symbol shard of the job
    text = workloads.generate(args.config, device=dev, seed=workloads.SEED + 101 * rank)
    builder = DeviceBuilder(dev)
    # c1's output is "8 packed bit vectors plus node borders" (BASELINE.json configs[0])
    want_borders = args.borders or args.config == "c1"
    outs = builder.alloc_outputs(n, sigma, want_borders)
    stream = torch.cuda.current_stream(dev)
    npass = len(pass_plan(n, sym_bytes, sigma, kind))

    def barrier():
        if world > 1:
            dist.barrier()

    sharded = world > 1
    transport = args.transport
    if sharded:
        from paper_1702_07578_b200.distributed import CudaOps, build_sharded

        ops = CudaOps(dev)
        if transport == "p2p":
            try:  # symmetric memory needs peer-accessible GPUs (NVLink); otherwise NCCL
                ops.peer_buffer(1)
            except Exception:  # noqa: BLE001
                transport = "nccl"
        ok = torch.tensor([1 if transport == "p2p" else 0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        transport = "p2p" if int(ok.item()) else "nccl"

    graphs = {}

    def one_build(kind_):
        if args.graph and not sharded:
            if kind_ not in graphs:
                graphs[kind_] = builder.capture(text, sigma, kind_, borders=want_borders)
            return graphs[kind_].replay()
        if sharded:
            # one WM/WT over the whole job's world * n symbols: local builds, NCCL
            # histogram all_gather, then the merge over peer memory (p2p) or the
            # bit-segment all_to_all + shift-merge (nccl)
            return build_sharded(text, sigma, kind_, ops=ops, transport=transport)
        return builder.build(text, sigma, kind_, outputs=outs, borders=want_borders, check=False)

    def timed(kind_, steps, warmup):
        for _ in range(warmup):
            one_build(kind_)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            one_build(kind_)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # correctness gate on the benchmark input: range status must be clean
    builder.build(text, sigma, kind, outputs=outs, borders=want_borders, check=True)
    launches_per_build = int(builder.lib.wvlt_last_launches())  # our kernels in one device build

    with ClockSampler(local) as clk:
        ms = timed(kind, args.steps, args.warmup)
    clocks = clk.summary()

    # per-stage profile (separate loop; events between stages)
    _lib.profile_enable(True)
    stage_ms: dict[str, list[float]] = {}
    for _ in range(max(3, min(args.steps, 5))):
        builder.build(text, sigma, kind, outputs=outs, borders=want_borders, check=False)
        for name, t in _lib.profile_read():
            stage_ms.setdefault(name, []).append(t)
    _lib.profile_enable(False)
    stages = {k: statistics.median(v) for k, v in stage_ms.items()}
    # the dominant kernel: the longest stage that moves the text (K1 or a level pass)
    dominant = max((k for k in stages if k == "hist" or k.startswith("pass")), key=lambda k: stages[k])
    peak, peak_src = peaks()
    mbytes = metric_bytes(n, sym_bytes, sigma)
    # SURVEY §8(d)'s per-unit figure (s + 1/8 bytes per symbol per level, s the
    # text's symbol bytes) times the units the dominant kernel processes per
    # launch (n symbols x the levels it emits), over its CUDA-event time
    dom_levels = stage_levels(dominant, n, sym_bytes, sigma, kind)
    dom_8d = dom_levels * (n * sym_bytes + 8 * ((n + 63) // 64))
    achieved = dom_8d / (stages[dominant] * 1e-3) / 1e9
    dom_bytes = stage_bytes(dominant, n, sym_bytes, sigma, kind)
    traffic = None
    tf = ROOT / "profiles" / f"ncu_traffic_{args.config}_{kind}.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(dominant)
    # the fused pass is not HBM-bound: its limiter comes from the same ncu capture
    # -- shared-memory wavefronts per SM per cycle of its CUDA-event duration at
    # the sampled clock, next to ncu's L1, issue-slot and ALU-pipe utilisation;
    # the busiest of these is reported as the resource
    limiter = None
    sf = ROOT / "profiles" / f"ncu_smem_{args.config}_{kind}.json"
    if sf.exists() and clocks.get("sm_mhz"):
        rec = json.loads(sf.read_text()).get(dominant)
        if isinstance(rec, (int, float)):
            rec = {"smem_wavefronts": rec}
        if rec and rec.get("smem_wavefronts"):
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            wf = rec["smem_wavefronts"]
            per_cycle = wf / (sms * stages[dominant] * 1e-3 * clocks["sm_mhz"] * 1e6)
            util = {"shared-memory pipe (wavefronts / SM / cycle)": per_cycle}
            if rec.get("issue_pct") is not None:
                util["instruction issue (ncu issue-active)"] = rec["issue_pct"] / 100
            if rec.get("l1_pct") is not None:
                util["L1 / shared-memory throughput (ncu)"] = rec["l1_pct"] / 100
            if rec.get("alu_pct") is not None:
                util["integer ALU pipe (ncu)"] = rec["alu_pct"] / 100
            res = max(util, key=util.get)
            limiter = {"resource": res, "frac": util[res], "utilisation": util, "wavefronts_per_launch": wf,
                       "inst_executed_per_launch": rec.get("inst_executed"),
                       "source": f"profiles/ncu_smem_{args.config}_{kind}.json (ncu --set full, one launch)"}

    value = world * n / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": {1: "u8", 2: "u16", 4: "u32"}[sym_bytes], "data": "synthetic",
        "config": {"workload": args.config, "description": workloads.DESCRIPTIONS[args.config], "kind": kind,
                   "n_per_gpu": n, "sigma": sigma, "levels": code_width(sigma), "passes": npass,
                   "l2": ("inputs larger than L2 (text %d MiB per GPU vs 126 MB L2); no flush" % (n * sym_bytes >> 20)
                          if n * sym_bytes > (126 << 20) else
                          "L2-resident input (text %d KiB); no flush: a launch-bound correctness config" % (n * sym_bytes >> 10)),
                   "graph": bool(args.graph and not sharded), "node_borders": bool(want_borders),
                   "parallelism": (f"sharded{world} (position shards; NCCL all_gather of histograms, "
                                   + ("merge over peer memory)" if transport == "p2p" else "NCCL all_to_all + merge)")
                                   if world > 1 else "single")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": dominant, "kernel_ms": stages[dominant],
                     "algorithmic_bytes": dom_8d, "levels": dom_levels,
                     "definition": "SURVEY 8d per-unit bytes (s + 1/8 per symbol per level) x the n symbols x levels "
                                   "the dominant kernel emits (its counting kernel emits the stage's first level), "
                                   "over its CUDA-event time",
                     "physical": {"bytes": traffic, "frac": (traffic / (stages[dominant] * 1e-3) / 1e9 / peak)
                                  if traffic else None, "kernel_own_bytes": dom_bytes,
                                  "kernel_own_frac": dom_bytes / (stages[dominant] * 1e-3) / 1e9 / peak,
                                  "note": "traffic = ncu dram bytes of one launch (profiles/); kernel_own_bytes = "
                                          "the text it reads + the bytes it writes"},
                     "peak_source": peak_src, "limiter": limiter},
        "metric_roofline": {"bytes_per_build": mbytes, "achieved_gbs": mbytes / (ms * 1e-3) / 1e9,
                            "frac": mbytes / (ms * 1e-3) / 1e9 / peak,
                            "frac_of_nominal_8tbs": mbytes / (ms * 1e-3) / 1e9 / 8000.0,
                            "definition": "SURVEY 8d: B = L (n s + n/8), text read once per level + level bits; "
                                          "frac against the measured copy peak, frac_of_nominal_8tbs against "
                                          "the 8 TB/s BASELINE.json names"},
        "stages_ms": stages,
        "clocks": clocks,
        "gpu_launches": args.steps * launches_per_build,
    }

    if not args.no_wt and kind == "wm":
        wt_ms = timed("wt", max(3, args.steps // 2), 2)
        line["wt"] = {"value": world * n / (wt_ms * 1e-3), "unit": UNIT, "ms_per_step": wt_ms,
                      "metric_roofline_frac": mbytes / (wt_ms * 1e-3) / 1e9 / peak}

    if not args.no_e2e:
        host = torch.empty(n, dtype=cfg["dtype"], pin_memory=True)
        host.copy_(text)
        w = code_width(sigma)
        nwords = (n + 63) // 64
        harr = host.numpy()
        e2e_steps = max(2, args.steps)
        # page-locked output buffers, used round robin by the builds of the queue
        hwords = [torch.empty((w, nwords), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
                  for _ in range(4)]
        builder.build_host(harr, sigma, kind, out_words=hwords[0])  # warm-up (device buffers, workspace)
        if not sharded:
            builder.build_host_batch([harr, harr], sigma, kind, out_words=hwords[:2])
        host_launches = int(builder.lib.wvlt_last_launches())
        torch.cuda.synchronize()

        lat_steps = max(2, min(args.steps, 5))
        if sharded:
            # N > 1: the job is the sharded global build -- every step each rank
            # uploads its shard, the ranks build and merge (build_sharded), and each
            # rank downloads the level words it owns; one step at a time (the merge
            # synchronises the ranks)
            dev_text = torch.empty_like(text)

            def e2e_step(hout=None):
                dev_text.copy_(host, non_blocking=True)
                res = build_sharded(dev_text, sigma, kind, ops=ops, transport=transport)
                if hout is None:
                    hout = torch.empty(res.level_words.shape, dtype=torch.int64, pin_memory=True)
                hout.copy_(res.level_words, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
                return hout

            try:
                hout = e2e_step()
                barrier()
                t0 = time.perf_counter()
                for _ in range(e2e_steps):
                    e2e_step(hout)
                dt = (time.perf_counter() - t0) / e2e_steps
            except Exception as ex:  # noqa: BLE001 - keep the device-resident line
                print(f"e2e (sharded) failed: {ex!r}", file=sys.stderr)
                dt = float("nan")
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
            hout = hout if dt == dt else torch.empty(0)
            line["e2e"] = {"value": world * n / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
                           "h2d_bytes_per_step": n * sym_bytes, "d2h_bytes_per_step": int(hout.numel()) * 8,
                           "steps": e2e_steps,
                           "path": f"per rank: H2D of its {n}-symbol shard from page-locked memory, build_sharded "
                                   f"({transport}), D2H of the level words it owns; bytes are per rank"}
            line["gpu_launches"] += e2e_steps * host_launches
            args.no_e2e = True  # the single-GPU queue below does not apply

    if not args.no_e2e:
        # latency: one build at a time through wvlt_build_host (H2D, build, D2H, sync)
        barrier()
        t0 = time.perf_counter()
        for _ in range(lat_steps):
            builder.build_host(harr, sigma, kind, out_words=hwords[0])
        lat = (time.perf_counter() - t0) / lat_steps

        # throughput: K builds as one queue through wvlt_build_host_batch -- the
        # upload of text i+1, the build of text i and the download of build i-1's
        # levels overlap (PCIe is full duplex); every build still moves its whole
        # text host->device and all its level words device->host inside the timed
        # region
        # three timed queues, the median reported (host-side hiccups of the copy
        # path -- an occasional one-off stall of a whole queue was seen -- do not
        # decide the figure)
        queue = [harr] * e2e_steps
        outs_q = [hwords[i % len(hwords)] for i in range(e2e_steps)]
        builder.build_host_batch(queue, sigma, kind, out_words=outs_q)  # warm-up at the timed queue length
        reps = []
        for _ in range(3):
            barrier()
            t0 = time.perf_counter()
            builder.build_host_batch(queue, sigma, kind, out_words=outs_q)
            reps.append((time.perf_counter() - t0) / e2e_steps)
        dt = statistics.median(reps)
        if world > 1:
            t = torch.tensor([dt, lat], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt, lat = float(t[0].item()), float(t[1].item())
        line["e2e"] = {"value": world * n / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
                       "h2d_bytes_per_step": n * sym_bytes,
                       "d2h_bytes_per_step": w * nwords * 8 + w * 8 + 4,
                       "steps": e2e_steps, "latency_ms": lat * 1e3,
                       "queues_ms_per_step": [round(r * 1e3, 3) for r in reps],
                       "path": "wvlt_build_host_batch (C ABI) over a queue of K builds with page-locked host "
                               "buffers: upload of text i+1, build i and download of build i-1's levels overlap "
                               "on three streams; latency_ms = one build at a time through wvlt_build_host"}
        line["gpu_launches"] += (lat_steps + e2e_steps) * host_launches

    if not args.no_api and not sharded and rank == 0:
        # the reference-facing Python API exactly as the reference's callers use it:
        # a pageable numpy text in, a WaveletMatrix / LevelWiseWaveletTree of
        # BitVectors (numpy words) out, node borders included
        import paper_1702_07578_b200 as wv

        arr = text.cpu().numpy()
        wv.build_structure(arr, sigma, kind, "ps")  # warm-up (staging buffers, workspace)
        api = []
        for _ in range(3):
            t0 = time.perf_counter()
            st = wv.build_structure(arr, sigma, kind, "ps")
            api.append(time.perf_counter() - t0)
            del st
        ta = statistics.median(api)
        line["e2e_api"] = {"value": n / ta, "unit": UNIT, "ms_per_step": ta * 1e3, "steps": len(api),
                           "h2d_bytes_per_step": n * sym_bytes, "d2h_bytes_per_step": code_width(sigma) * ((n + 63) // 64) * 8,
                           "path": "paper_1702_07578_b200.build_structure(numpy text, sigma, kind, 'ps') -> "
                                   "structure of BitVectors (pageable numpy in and out, node borders included), "
                                   "one call at a time, median of 3"}

    if not args.no_cpu and rank == 0:
        sample = min(n, args.cpu_sample) if args.cpu_sample else n
        host_np = text[:sample].cpu().numpy()
        line["cpu_baseline"] = cpu_baseline(host_np, sigma, kind, sample)
        line["cpu_baseline"].pop("seconds_per_build", None)

    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
