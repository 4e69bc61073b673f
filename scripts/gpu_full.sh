mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 900 -x -rf > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_full.log
for c in 1 0 2 3 4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.log; echo "cfg$c rc=$?"; done
