mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x -k "batch or estimator or bins or golden or errors or empty or reversal or cli" > gpurun_out/api_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/api_tests.log
python scripts/api_bench.py 10 > gpurun_out/api_bench.json; cat gpurun_out/api_bench.json
