"""Key metrics + SASS hot spots of an ncu report: python scripts/ncu_summary.py rep [top]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
keys = ("Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy",
        "Executed Instructions", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size",
        "Block Size", "Dynamic Shared Memory Per Block", "Block Limit Registers",
        "Block Limit Shared Mem")
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
for row in csv.reader(io.StringIO(out)):
    while row and row[-1] == "":
        row = row[:-1]
    if len(row) > 3 and row[-3] in keys:
        print(f"{row[-3]:40s} {row[-1]:>14} {row[-2]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if len(rows) > 2:
    hdr, units, vals = rows[0], rows[1], rows[2]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                 "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
        if name in hdr:
            i = hdr.index(name)
            print(f"{name:60s} {vals[i]:>16} {units[i]}")
if top:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr, data = rows[1], rows[2:]
    ie, sc, ws = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    tot = sum(float(r[ie] or 0) for r in data)
    st = sum(float(r[ws] or 0) for r in data)
    print(f"instructions {tot:.3e}, stall samples {st:.0f}")
    for r in sorted(data, key=lambda r: -float(r[ws] or 0))[:top]:
        print(f"{r[0][-5:]} inst={float(r[ie] or 0) / tot * 100:5.2f}% "
              f"stall={float(r[ws] or 0) / st * 100:5.2f}%  {r[sc][:70]}")
