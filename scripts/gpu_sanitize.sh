# NOTE: compute-sanitizer is closed on the shared GPU pool (it left GPUs needing resets);
# bounds are checked instead by guard-band tests (tests/test_gpu_property.py).
# compute-sanitizer memcheck / racecheck / synccheck over a parity subset (small inputs)
mkdir -p gpurun_out
SEL="(golden or window_search or bins_vs or odd_shapes or overflow or cfg0_full or pipeline_matches or pipeline_back or pipeline_edge or generic or slot_width or many_channels or fused_cta or unaligned) and not binned"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -2
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_reversal.py -q -m gpu -x -k "device_descent or batched or matches_reference" -p no:cacheprovider \
  > gpurun_out/sanitize_reversal.log 2>&1
echo "reversal memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_reversal.log | tail -2
