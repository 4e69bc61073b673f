mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "slab_pair or bins or overflow or many_channels" > gpurun_out/items_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/items_tests.log
CFGS="3" bash scripts/gpu_ab_env.sh "VG_ITEMS=0" "VG_ITEMS=1" "VG_ITEMS=1 VG_PLAN_Q=4" "VG_ITEMS=1 VG_TASK_KB=256"
