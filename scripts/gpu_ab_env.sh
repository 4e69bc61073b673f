# A/B of environment settings: gpu_ab_env.sh "VG_SW=4" "VG_SW=8" ...
mkdir -p gpurun_out
for setting in "$@"; do
  for c in ${CFGS:-1 4 3 2}; do
    env $setting timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abenv.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/abenv.json')); print('AB $setting', $c, round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['k3_ms'],4), round(d['roofline']['k1_ms'],4))"
  done
done
