mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "slab_pair" > gpurun_out/yp_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/yp_tests.log
CFGS="1 4 3 2" bash scripts/gpu_ab_env.sh "VG_YP=1" "VG_YP=2"
