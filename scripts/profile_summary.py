"""Write profiles/<tag>_*.txt summaries from an ncu report + launch list.

usage: python scripts/profile_summary.py <tag> <report.ncu-rep> [launches.csv]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

tag, rep = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else None
out = Path("profiles")
out.mkdir(exist_ok=True)

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy",
        "Executed Instructions", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "No Eligible", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block", "SM Frequency", "DRAM Frequency", "Compute (SM) Throughput")
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
lines = [f"# ncu --set full summary ({rep}); --clock-control none"]
by_kernel = {}
for row in csv.reader(io.StringIO(det)):
    while row and row[-1] == "":
        row = row[:-1]
    if len(row) > 5 and row[-3] in KEYS:
        by_kernel.setdefault((row[0], row[4]), []).append(f"  {row[-3]:38s} {row[-1]:>16} {row[-2]}")
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
traffic = {}
for (kid, kname), items in by_kernel.items():
    lines.append(f"\n== launch {kid}: {kname}")
    lines += items
    for r in rows[2:]:
        if r[hdr.index("ID")] == kid:
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                      "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                      "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                      "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                      "sm__warps_active.avg.pct_of_peak_sustained_active"):
                if m in hdr:
                    i = hdr.index(m)
                    lines.append(f"  {m:60s} {r[i]:>14} {units[i]}")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(m)
                b += float(r[i]) * scale[units[i]]
            traffic[kname] = b
(out / f"{tag}_ncu_summary.txt").write_text("\n".join(lines) + "\n")
if launches:
    rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    txt = ["# per-launch device time (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)",
           "kernel,ns"]
    for r in rows[1:]:
        txt.append(f"{r[ki][:70]},{r[vi]}")
    (out / f"{tag}_launches.csv").write_text("\n".join(txt) + "\n")
print(json.dumps(traffic))
