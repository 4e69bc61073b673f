"""Group SASS of an ncu report into equal-count blocks; print the heaviest."""
import csv, io, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
ie, sc, ws = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ie] or 0) for r in data); st = sum(float(r[ws] or 0) for r in data) or 1
blocks, cur = [], None
for r in data:
    v, w = float(r[ie] or 0), float(r[ws] or 0)
    if cur and abs(cur[1] - v) < 1e-9:
        cur[2] += 1; cur[3] += w; cur[4].append(r[sc].strip()[:44])
    else:
        cur = [r[0][-5:], v, 1, w, [r[sc].strip()[:44]]]; blocks.append(cur)
print(f"total {tot:.4e} instructions")
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:top]:
    print(f"{b[0]} count={b[1]:.3e} n={b[2]:3d} share={b[1]*b[2]/tot*100:5.1f}% stall={b[3]/st*100:5.1f}%  {b[4][0]} | {b[4][-1]}")
if len(sys.argv) > 3:
    on = False
    for r in data:
        if r[0][-5:] == sys.argv[3]: on = True
        if on:
            print(r[0][-5:], r[ie], r[sc][:90])
            if r[0][-5:] == sys.argv[4]: break
