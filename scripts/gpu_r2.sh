#!/usr/bin/env bash
# Round-2 check on one B200: smoke, full GPU suite, default bench line, the
# self-spawned 2-rank bench (ranks share cuda:0, gloo plumbing), the reference
# arm, and the launch list of the bench command.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests/ -q -m gpu --timeout 900 -rf ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_full.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo "bench rc=$?"; cat gpurun_out/bench_default.json
timeout 600 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.log; echo "bench g2 rc=$?"; cat gpurun_out/bench_g2.json; tail -3 gpurun_out/bench_g2.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
[ "${NO_PROFILE:-0}" = 1 ] || bash scripts/gpu_profile.sh
