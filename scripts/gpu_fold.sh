mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "slab_pair or cfg4 or many_channels or fused_cta or pipeline" > gpurun_out/fold_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fold_tests.log
R=3 CFGS="4 1" bash scripts/gpu_abr.sh libvg_base.so libvoxgrid_b200.so
