# A/B of library builds: bench cfg1/3/4 per variant (VG_LIB), plus VG_ZW variants
mkdir -p gpurun_out
for lib in "$@"; do
  for c in ${CFGS:-1 4 3}; do
    VG_LIB=$PWD/paper_2211_08506_b200/$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${lib}_cfg$c.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/ab_${lib}_cfg$c.json')); print('$lib', $c, round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['k3_ms'],4))"
  done
done
