mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reversal.py tests/test_io_cli.py -q -m gpu -x > gpurun_out/rev_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rev_tests.log
python scripts/reversal_bench.py gpu 4 200 > gpurun_out/rev_gpu.json; cat gpurun_out/rev_gpu.json | head -c 300; echo
python scripts/reversal_bench.py gpu-batch 4 200 > gpurun_out/rev_gpu_b4.json; cat gpurun_out/rev_gpu_b4.json | head -c 300; echo
python scripts/reversal_bench.py gpu-batch 64 200 > gpurun_out/rev_gpu_b64.json; cat gpurun_out/rev_gpu_b64.json | head -c 300; echo
