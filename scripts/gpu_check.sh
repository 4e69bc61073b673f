mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
python -c "import numpy.lib.introspect as i; print(i.opt_func_info(func_name='exp', signature='float32'))"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -p pytest_timeout --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -40 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.log; echo "bench rc=$?"; cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.log
