mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 900 -rf > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/gpu_tests.log
CMD="python bench.py --steps 3 --warmup 3 --batch 256 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:vg_slab_kernel -s 4 -c 1 -o gpurun_out/prof_k3 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
