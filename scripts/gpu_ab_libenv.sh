# A/B of (library, environment) pairs: gpu_ab_libenv.sh "libv_x.so|VG_A=1 VG_B=2" ...
mkdir -p gpurun_out
for pair in "$@"; do
  lib="${pair%%|*}"; setting="${pair#*|}"
  for c in ${CFGS:-1 4 3 2}; do
    env VG_LIB=$PWD/paper_2211_08506_b200/$lib $setting timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ablib.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ablib.json')); print('AB $lib $setting', $c, round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['k3_ms'],4))"
  done
done
