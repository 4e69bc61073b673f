# Full GPU suite + smoke (round-end check)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 900 -rf > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_full.log
