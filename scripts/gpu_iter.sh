# quick iteration: parity subset + bench + optional ncu (arg1 = "ncu")
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 600 -x -k "golden or cfg0 or cfg1 or odd or overflow or empty or generic" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench rc=$?"; cat gpurun_out/bench.json
if [ "$1" = "ncu" ]; then
CMD="python bench.py --steps 3 --warmup 3 --batch 256 --no-cpu-baseline"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:vg_slab -s 4 -c 1 -o gpurun_out/prof_k3 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_full.log
fi
