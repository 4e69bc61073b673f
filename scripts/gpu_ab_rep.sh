# Repeated A/B of environment settings on one config: CFG=3 REPS=3 STEPS=30 gpu_ab_rep.sh "VG_A=1" ...
mkdir -p gpurun_out
for r in $(seq ${REPS:-3}); do
  for setting in "$@"; do
    env $setting timeout 300 python bench.py --config ${CFG:-3} --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline > gpurun_out/abrep.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('gpurun_out/abrep.json')); print('AB $setting', ${CFG:-3}, round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['k3_ms'],4))"
  done
done
