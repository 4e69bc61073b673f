"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills, stack, smem."""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "paper_2211_08506_b200/csrc/vg_kernels.cu"
cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
       "-fmad=false", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared",
       "-Iinclude", "-o", "/tmp/_ptxas.so", src]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
if "error" in out:
    print(out)
    sys.exit(1)
cur = None
for line in out.splitlines():
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        name = re.sub(r"_ZN\d+_(GLOBAL|INTERNAL)\w*?_cu_\w{8}\d*", "", cur)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        stack, ss, sl = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        sm = re.search(r"(\d+) bytes smem", line)
        print(f"{name[:70]:70s} regs={m.group(1):>3} spill={ss:>3}/{sl:>3} stack={stack:>3} "
              f"smem={sm.group(1) if sm else 0}")
        cur = None
