mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused_halving or many_channels or cfg4 or cfg0 or pipeline or slab_pair or golden" > gpurun_out/fh_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fh_tests.log
R=3 CFGS="4 1" bash scripts/gpu_abr.sh libvg_base.so libvoxgrid_b200.so
