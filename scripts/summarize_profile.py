"""Turn one gpurun_out/ round of GPU evidence into tracked files under profiles/.

  python scripts/summarize_profile.py <tag> <node_updates_in_profiled_launch>

reads   gpurun_out/bench_<tag>.log        (bench.py JSON line, no profiler)
        gpurun_out/launches_<tag>.csv     (ncu --metrics gpu__time_duration.sum launch list)
        gpurun_out/prof_<tag>.ncu-rep     (ncu --set full of one K1 launch)
writes  profiles/bench_<tag>.json, profiles/launches_<tag>.csv,
        profiles/ncu_K1_<tag>.txt (pipe utilisation, issue, LSU, DRAM, stalls,
        SASS instruction mix per node-update)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
nu = float(sys.argv[2]) if len(sys.argv) > 2 else None
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)

# bench line
b = os.path.join(G, f"bench_{tag}.log")
if os.path.exists(b):
    lines = [ln for ln in open(b) if ln.startswith("{")]
    if lines:
        with open(os.path.join(P, f"bench_{tag}.json"), "w") as f:
            f.write(lines[-1])

# launch list (kernel, block, grid, ns) + share of the step
lpath = os.path.join(G, f"launches_{tag}.csv")
if os.path.exists(lpath):
    rows = [r for r in csv.reader(open(lpath)) if len(r) > 10 and r[0] != "ID"]
    tot = sum(float(r[-1]) for r in rows)
    # share of the dominant trajectory kernel (K1b bitslice_kernel or K1 traj_kernel)
    top = "bitslice_kernel" if any("bitslice_kernel" in r[4] for r in rows) else "traj_kernel"
    k1 = sum(float(r[-1]) for r in rows if top in r[4])
    with open(os.path.join(P, f"launches_{tag}.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "block", "grid", "gpu_time_ns"])
        for r in rows:
            w.writerow([r[4][:90], r[7], r[8], r[-1]])
        w.writerow([f"# {top} share of all launched GPU time: {k1 / tot:.6f}", "", "", ""])

rep = os.path.join(G, f"prof_{tag}.ncu-rep")
if not os.path.exists(rep):
    sys.exit(0)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
out = io.StringIO()
kname = get.get('Kernel Name', ('', '?'))[1]
kshort = "K1b" if "bitslice" in kname else "K1"
out.write(f"ncu --set full --clock-control none, one {kshort} launch, tag {tag}\n")
out.write(f"kernel: {kname}\n\n")
keys = ["gpu__time_duration.sum", "sm__cycles_active.avg", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum"]
for k in keys:
    if k in get:
        out.write(f"{k:80s} {get[k][0]:10s} {get[k][1]}\n")
out.write("\nwarp stall reasons (per issue-active, ratio):\n")
st = []
for h, (u, v) in get.items():
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for v, h in sorted(st, reverse=True)[:12]:
    out.write(f"  {h:30s} {v:.3f}\n")

# SASS instruction mix
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
if len(srows) > 2:
    sh = srows[1]
    ie, sc = sh.index("Instructions Executed"), sh.index("Source")
    c = Counter()
    tot = 0
    for r in srows[2:]:
        if not r[ie].isdigit():
            continue
        n = int(r[ie])
        t = r[sc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        c[op] += n
        tot += n
    out.write(f"\nSASS warp-instructions executed: {tot}\n")
    if nu:
        out.write(f"node-updates in the profiled launch: {nu:.6g}; "
                  f"thread-instructions per node-update = warp-inst x 32 / node-updates = {tot * 32 / nu:.2f}\n")
    out.write("top opcodes (warp-instructions x 32 per node-update):\n")
    for k, v in c.most_common(28):
        out.write(f"  {k:26s} {v * 32 / nu if nu else v:8.2f}\n")
with open(os.path.join(P, f"ncu_{kshort}_{tag}.txt"), "w") as f:
    f.write(out.getvalue())
print(out.getvalue())
