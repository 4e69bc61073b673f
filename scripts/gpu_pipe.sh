mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "pipeline or golden or cfg0" > gpurun_out/pipe_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pipe_tests.log
timeout 120 python scripts/pipe_overhead.py
for c in 0 1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.log; echo "cfg$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_cfg$c.json')); print($c, round(d['value']), round(d['value_serial']), round(d['e2e']['value']), d['e2e']['ms_per_step_event'], d['e2e']['ms_per_step_wall'], round(d['roofline']['frac'],3))"; done
