# compute-sanitizer memcheck / racecheck / synccheck over a parity subset (small inputs)
mkdir -p gpurun_out
SEL="golden or window_search or bins or odd_shapes or overflow or cfg0_full or pipeline or generic or slot_width"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -2
done
