mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "slab_pair or golden or overflow or many_channels or cfg0 or dense" > gpurun_out/nz_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/nz_tests.log
CFGS="3 4 1 2" bash scripts/gpu_ab.sh libvg_base.so libvoxgrid_b200.so
