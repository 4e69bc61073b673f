#!/usr/bin/env bash
# ncu --set full of K1 (vg_tables_open_kernel) at one config: gpu_k1prof_cfg.sh <config> <batch>
mkdir -p gpurun_out
CMD="python bench.py --config $1 --batch $2 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/k1_plain_$1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:vg_tables_open -s 3 -c 1 \
  -o gpurun_out/prof_k1_cfg$1 -f $CMD > gpurun_out/ncu_k1_$1.log 2>&1; echo "k1 ncu cfg$1 rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_k1_cfg$1.ncu-rep > gpurun_out/k1_cfg$1_summary.txt 2>&1
python scripts/ncu_lines.py gpurun_out/prof_k1_cfg$1.ncu-rep 25 > gpurun_out/k1_cfg$1_lines.txt 2>&1
ncu -i gpurun_out/prof_k1_cfg$1.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin))
for h, u, v in zip(rows[0], rows[1], rows[2]):
    if 'average_warps_issue_stalled' in h and 'per_issue_active' in h and float(v or 0) > 0.05:
        print(h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), v)
" > gpurun_out/k1_cfg$1_stalls.txt
