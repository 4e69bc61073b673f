mkdir -p gpurun_out
timeout 900 python -m paper_2211_08506_b200 bench --output gpurun_out/protocol_gpu_full.json > gpurun_out/protocol_gpu_full.log 2>&1; echo "full rc=$?"
timeout 900 python -m paper_2211_08506_b200 bench --sizes 16,32,64 --repeats 2 --molecules 100 --output gpurun_out/protocol_gpu_small.json > gpurun_out/protocol_gpu_small.log 2>&1; echo "small rc=$?"
tail -30 gpurun_out/protocol_gpu_full.log
