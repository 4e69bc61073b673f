# ncu --set full of K1+K3 for one config: gpu_prof_cfg.sh <config> <batch> <tag>
mkdir -p gpurun_out
CMD="python bench.py --config $1 --batch $2 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_$3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${4:-vg_slab|vg_tables}" -s ${5:-6} -c ${6:-2} -o gpurun_out/prof_$3 -f $CMD > gpurun_out/ncu_$3.log 2>&1; echo "ncu $3 rc=$?"
