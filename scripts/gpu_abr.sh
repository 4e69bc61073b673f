# Interleaved A/B of library builds (R rounds, median per build and config):
# R=3 CFGS="3 4" bash scripts/gpu_abr.sh libA.so libB.so [ENVSPEC...]
# A build may carry env settings: "libvoxgrid_b200.so:VG_BULK=0"
mkdir -p gpurun_out
rm -f gpurun_out/abr.txt
for r in $(seq ${R:-3}); do
  for spec in "$@"; do
    lib=${spec%%:*}; envs=""; [ "$spec" != "$lib" ] && envs=${spec#*:}
    for c in ${CFGS:-1 4 3}; do
      env $envs VG_LIB=$PWD/paper_2211_08506_b200/$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abr.json 2>/dev/null
      python -c "import json; d=json.load(open('gpurun_out/abr.json')); print('$spec', $c, d['roofline']['k3_ms'], d['roofline']['frac'], d['value'])" >> gpurun_out/abr.txt
    done
  done
done
python - <<'PY'
import collections, statistics
d = collections.defaultdict(list)
for line in open("gpurun_out/abr.txt"):
    spec, c, k3, frac, val = line.split()
    d[(spec, c)].append((float(k3), float(frac), float(val)))
for (spec, c), v in sorted(d.items(), key=lambda kv: (kv[0][1], kv[0][0])):
    k3 = statistics.median(x[0] for x in v); fr = statistics.median(x[1] for x in v)
    print(f"ABR cfg{c} {spec:40s} k3 {k3:.4f} ms  frac {fr:.3f}  (n={len(v)}, k3 range {min(x[0] for x in v):.4f}-{max(x[0] for x in v):.4f})")
PY
