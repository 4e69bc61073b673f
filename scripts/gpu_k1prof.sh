#!/usr/bin/env bash
# ncu --set full of K1 (vg_tables_open_kernel) at the bench workload (cfg1):
# FP32 / FP64 / XU (SFU) pipe utilisation for the compute leg of the roofline.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/k1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:vg_tables_open -s 3 -c 1 \
  -o gpurun_out/prof_k1_cfg1 -f $CMD > gpurun_out/ncu_k1.log 2>&1; echo "k1 ncu rc=$?"
ncu -i gpurun_out/prof_k1_cfg1.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin))
hdr, units, vals = rows[0], rows[1], rows[2]
for h, u, v in zip(hdr, units, vals):
    if any(k in h for k in ('pipe_xu', 'pipe_fma', 'pipe_fp64', 'pipe_alu', 'inst_executed.sum', 'gpu__time_duration.sum', 'sm__throughput', 'dram__bytes', 'issue_active', 'pipe_fp16', 'inst_executed_pipe')):
        print(h, u, v)
" > gpurun_out/k1_pipes.txt; wc -l gpurun_out/k1_pipes.txt
