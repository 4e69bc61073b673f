"""Per-CUDA-source-line instructions and stall samples of an ncu report:
python scripts/ncu_lines.py rep [top] [kernel regex]  (needs -lineinfo builds)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilter = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kfilter, "--page", "source", "--csv",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows:
    if r and r[0].isdigit():
        # source text may carry unescaped quotes: index the metrics from the end
        v = lambda i: float(r[len(r) - len(hdr) + i]) if r[len(r) - len(hdr) + i] not in ("", "-") else 0.0
        lines.append((int(r[0]), r[1].strip(), v(ie), v(ws)))
ti = sum(l[2] for l in lines) or 1
ts = sum(l[3] for l in lines) or 1
print(f"instructions {ti:.3e}  stall samples {ts:.0f}")
for ln, src, i, s in sorted(lines, key=lambda l: -(l[2] / ti + l[3] / ts))[:top]:
    print(f"{ln:5d} inst={i / ti * 100:5.1f}% stall={s / ts * 100:5.1f}%  {src[:90]}")
