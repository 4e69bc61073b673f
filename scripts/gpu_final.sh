#!/usr/bin/env bash
# Round-end evidence on one B200: smoke, full GPU suite, bench lines of every
# config, shard-sized batches (strong-scaling projection), 2-rank self-spawn,
# reference arm, launch list + ncu --set full of cfg1 and cfg3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests/ -q -m gpu --timeout 900 -rf > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_full.log
timeout 600 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.log; echo "bench rc=$?"
for c in 0 2 3 4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.log; echo "cfg$c rc=$?"; done
for b in 512 256 128; do timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_shard$b.json 2>/dev/null; echo "shard$b rc=$?"; done
timeout 600 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.log; echo "bench g2 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"
bash scripts/gpu_profile.sh
bash scripts/gpu_prof_cfg.sh 3 32 cfg3 "vg_slab_kernel" 3 1
