"""Summarize a round's ncu captures into profiles/ (run in the build container).

    python tools/summarize_profiles.py r1
Reads gpurun_out/launches_<tag>.csv (launch list) and gpurun_out/full_<tag>.ncu-rep
(--set full capture) and writes profiles/<tag>_launches.csv (trimmed),
profiles/<tag>_summary.md and profiles/ncu_traffic_c2_wm.json.
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = ROOT / "profiles"
out.mkdir(exist_ok=True)


def short(name):
    for k in ("hist8_kernel", "tiles8_kernel", "level_pass8q_kernel", "level_pass8_kernel", "scan8_chunks_kernel", "scan8_carry_kernel",
              "scan8_apply_kernel", "tables8_kernel",
              "hist_u8_kernel", "hist_generic_kernel", "digits_fast_kernel", "digits_kernel", "wm_pass_tables_kernel", "tables_kernel", "scan_reduce_kernel",
              "scan_apply_kernel", "level_pass_u8_kernel", "level_pass_kernel", "merge_bits_kernel", "widen_kernel"):
        i = name.find(k)
        if i >= 0:
            rest = name[i + len(k):]
            return k + (rest[:rest.index(">") + 1] if rest.startswith("<") else "")
    return "torch:" + name.split("(")[0].replace("void ", "")[-48:]


# ---- launch list ----
rows = list(csv.reader(open(ROOT / "gpurun_out" / f"launches_{tag}.csv")))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
launches = [(short(r[ki]), float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
with open(out / f"{tag}_launches.csv", "w") as f:
    f.write("kernel,duration_ns\n")
    for k, v in launches:
        f.write(f"{k},{v:.0f}\n")
# per-build breakdown: the bench does warm-up + timed builds of identical launches
tot = collections.defaultdict(float)
cnt = collections.Counter()
for k, v in launches:
    tot[k] += v
    cnt[k] += 1
grand = sum(tot.values())

# ---- full capture ----
raw = subprocess.run(["ncu", "-i", str(ROOT / "gpurun_out" / f"full_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active"]
units = rr[1]
full = []
for r in rr[2:]:
    full.append({w: r[h.index(w)] for w in want if w in h})


def mb(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}.get(unit, 1.0)


lines = [f"# Profile summary, round tag `{tag}` (c2: WM, n=2^30 uint8, sigma=256, Zipf 1.1)", "",
         "Source: `tools/profile_round.sh` under gpurun on one B200; `ncu` numbers are cold-cache and",
         "serialised, so compare shares, not absolute times, with bench.py's CUDA-event stages.", "",
         "## Launch list share (ncu gpu__time_duration.sum over all launches of the bench command)", "",
         "Torch kernels are the benchmark's synthetic-input generator (outside the timed region).", "",
         "| kernel | launches | total ms | share |", "|---|---|---|---|"]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    lines.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {100 * v / grand:.1f}% |")
lines += ["", "## `--set full` capture of the top kernels (one launch each)", "",
          "| kernel | time us | DRAM read MB | DRAM write MB | DRAM %peak | SM %peak | issue % | ALU % | LSU % | L1 %peak | smem wavefronts | bank conflicts | regs |",
          "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
smem = {}
ui = {w: units[h.index(w)] for w in want if w in h}
pass_idx = 0
for r in full:
    name = short(r["Kernel Name"])
    t_us = float(r["gpu__time_duration.sum"].replace(",", "")) * ({"us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}.get(ui["gpu__time_duration.sum"], 1))
    rd = mb(r["dram__bytes_read.sum"], ui["dram__bytes_read.sum"])
    wr = mb(r["dram__bytes_write.sum"], ui["dram__bytes_write.sum"])
    lines.append(f"| `{name}` | {t_us:.1f} | {rd:.1f} | {wr:.1f} | {r['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']} | "
                 f"{r['sm__throughput.avg.pct_of_peak_sustained_elapsed']} | {r['smsp__issue_active.avg.pct_of_peak_sustained_active']} | "
                 f"{r['sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active']} | {r['sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']} | "
                 f"{r.get('l1tex__throughput.avg.pct_of_peak_sustained_active', '')} | "
                 f"{r['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']} | {r['l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']} | {r['launch__registers_per_thread']} |")
    if "level_pass" in name:
        traffic[f"pass{pass_idx}"] = (rd + wr) * 1e6
        fnum = lambda k: float(r[k].replace(",", "")) if r.get(k) not in (None, "", "n/a") else None
        smem[f"pass{pass_idx}"] = {"smem_wavefronts": fnum("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                                   "l1_pct": fnum("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                                   "issue_pct": fnum("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                   "alu_pct": fnum("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                                   "inst_executed": fnum("smsp__inst_executed.sum")}
        pass_idx += 1
    elif "hist" in name or "digits" in name:
        traffic["hist"] = (rd + wr) * 1e6
    elif "tiles8" in name:
        traffic["tiles8"] = (rd + wr) * 1e6
(out / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
json.dump(traffic, open(out / "ncu_traffic_c2_wm.json", "w"), indent=1)
json.dump(smem, open(out / "ncu_smem_c2_wm.json", "w"), indent=1)  # per launch: smem wavefronts, L1 / issue / ALU utilisation
print("\n".join(lines))
print(traffic)
