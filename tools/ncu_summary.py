"""Key counters of the first kernel in an ncu report (raw page): time, instructions,
shared-memory wavefronts, pipe utilisation and the main stall reasons.

    python tools/ncu_summary.py report.ncu-rep [more reports ...]
"""
import csv
import subprocess
import sys

KEYS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6),
    ("inst_M", "smsp__inst_executed.sum", 1e-6),
    ("smem_wf_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
    ("smem_st_wf_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", 1e-6),
    ("smem_ld_wf_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 1e-6),
    ("l1_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("alu_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("fma_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    ("lsu_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("xu_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("regs", "launch__registers_per_thread", 1),
]
STALLS = ["barrier", "mio_throttle", "short_scoreboard", "long_scoreboard", "wait", "math_pipe_throttle",
          "not_selected", "lg_throttle", "dispatch_stall", "branch_resolving"]

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2]
    get = lambda k: float(v[h.index(k)].replace(",", "")) if k in h and v[h.index(k)] not in ("", "n/a") else float("nan")
    print(f"== {rep}: {v[h.index('Kernel Name')][:70]}")
    print("  " + "  ".join(f"{n}={get(k) * s:.3g}" for n, k, s in KEYS))
    st = {s: get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio") for s in STALLS}
    print("  stalls/issue: " + "  ".join(f"{k}={x:.2f}" for k, x in sorted(st.items(), key=lambda kv: -kv[1])))
