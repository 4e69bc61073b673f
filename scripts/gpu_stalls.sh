# warp stall-reason breakdown of K3 at one config: gpu_stalls.sh <config> <batch>
mkdir -p gpurun_out
CMD="python bench.py --config $1 --batch $2 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --metrics regex:smsp__average_warps_issue_stalled_.*_per_issue_active.ratio --clock-control none -k regex:vg_slab -s 2 -c 1 --csv $CMD > gpurun_out/stalls_cfg$1.csv 2>&1; echo "rc=$?"
