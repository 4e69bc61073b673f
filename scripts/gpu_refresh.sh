# Round-end evidence: bench lines for every config, reference arm, launch
# list + ncu --set full of the bench workload (cfg1, report kept), and full
# captures of K3 at cfg3 / cfg4 summarised on the box (reports dropped: the
# copy-back limit is 64 MiB). Run the GPU tests separately (gpu_tests.sh).
mkdir -p gpurun_out/sum
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"
for c in 0 2 3 4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.log; echo "cfg$c rc=$?"; done
bash scripts/gpu_profile.sh
for c in 3 4; do
  b=$([ $c = 3 ] && echo 32 || echo 4096)
  bash scripts/gpu_prof_cfg.sh $c $b cfg$c vg_slab 2 1
  (cd gpurun_out/sum && python ../../scripts/profile_summary.py cfg$c ../prof_cfg$c.ncu-rep > /dev/null)
  python scripts/ncu_lines.py gpurun_out/prof_cfg$c.ncu-rep 40 > gpurun_out/sum/cfg${c}_lines.txt 2>&1
  python scripts/sass_blocks.py gpurun_out/prof_cfg$c.ncu-rep 12 > gpurun_out/sum/cfg${c}_sass.txt 2>&1
  rm -f gpurun_out/prof_cfg$c.ncu-rep
done
ls -la gpurun_out gpurun_out/sum
