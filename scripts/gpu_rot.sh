mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "slab_pair or bins or overflow" > gpurun_out/rot_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rot_tests.log
R=3 CFGS="3 4" bash scripts/gpu_abr.sh libvg_base.so libvoxgrid_b200.so
