# Launch list + one full ncu capture of K1 and K3 at the bench's default workload (cfg1).
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"vg_slab_kernel|vg_tables" -s 6 -c 2 -o gpurun_out/prof_cfg1 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/ncu_full.log
