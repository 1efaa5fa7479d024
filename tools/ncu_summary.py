"""Key metrics of every kernel in an ncu report (details page).  usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Executed Instructions", "Grid Size",
        "Block Size", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, ii, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
seen = {}
for r in rows[1:]:
    if r[mi] in WANT:
        key = (r[ii], r[ki].split("(")[0][:60])
        seen.setdefault(key, []).append(f"{r[mi]}={r[vi]} {r[ui]}".strip())
for (i, k), vals in seen.items():
    print(f"[{i}] {k}")
    for v in vals:
        print("     ", v)
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
cols = [c for c in h if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                              "sm__inst_executed_pipe_fma.sum", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active")]
for r in rr[2:]:
    print(r[h.index("Kernel Name")][:40], {c: r[h.index(c)] + " " + rr[1][h.index(c)] for c in cols})
