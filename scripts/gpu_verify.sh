mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 900 -x -rf > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_full.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo "bench rc=$?"; cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
for c in 0 2 3 4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.log; echo "cfg$c rc=$?"; done
