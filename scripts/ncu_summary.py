"""Summarise an ncu report: pipe utilisation, LSU wavefronts, stalls, per-opcode counts."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__cycles_active.avg", "smsp__cycles_active.avg"]
for h, u, v in zip(hdr, units, vals):
    if h in want or ("pipe" in h and "pct_of_peak_sustained_active" in h and "inst_executed" in h):
        print(f"{h:80s} {u:8s} {v}")
for h, u, v in zip(hdr, units, vals):
    if h.startswith("smsp__average_warp_latency_issue_stalled") or h.startswith("smsp__pcsamp_warps_issue_stalled"):
        try:
            if float(v) > 0.02 * 1:
                print(f"{h:80s} {u:8s} {v}")
        except ValueError:
            pass
