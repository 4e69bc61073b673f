mkdir -p gpurun_out
for c in 3 1 4; do VG_LIB=$PWD/paper_2211_08506_b200/libvg_timing.so timeout 300 python scripts/cta_timing.py $c gpurun_out/ts_cfg$c.npy; done
