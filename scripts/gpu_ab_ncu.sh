# ncu --set full of K3 for several library builds (VG_LIB), cfg1 batch 256
mkdir -p gpurun_out
for lib in "$@"; do
  CMD="python bench.py --steps 3 --warmup 3 --batch 256 --no-cpu-baseline"
  VG_LIB=$PWD/paper_2211_08506_b200/$lib $CMD > gpurun_out/plain_$lib.log 2>&1 && \
  VG_LIB=$PWD/paper_2211_08506_b200/$lib ncu --set full --clock-control none --import-source on -k regex:vg_slab -s 4 -c 1 -o gpurun_out/ab_$lib -f $CMD > gpurun_out/ncu_$lib.log 2>&1; echo "$lib ncu rc=$?"
done
