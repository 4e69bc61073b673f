"""Descent cost of grid reversal: refine_coords from the
detected peaks of cfg0 molecules for a fixed iteration budget.

  python scripts/reversal_bench.py gpu  [n_molecules] [iters]   # this repo, on cuda:0
  python scripts/reversal_bench.py gpu-batch [n] [iters]        # all n descents batched
  python scripts/reversal_bench.py reference [n] [iters]        # voxgrid (needs /root/reference)

Prints one JSON line: iterations/s and ms per iteration over the sample (the
reference evaluates backoff candidates one at a time; the GPU path evaluates
all 11 in one batched launch and keeps the reference's choice rule)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2211_08506_b200 import synth  # noqa: E402

impl = sys.argv[1]
n_mol = int(sys.argv[2]) if len(sys.argv) > 2 else 4
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cfg = synth.CONFIGS[0]

if impl == "reference":
    sys.path.insert(0, "/root/reference/pkg/src")
    import voxgrid as vg  # noqa: E402
    from voxgrid import reversal as rv  # noqa: E402
else:
    import paper_2211_08506_b200 as vg  # noqa: E402
    from paper_2211_08506_b200 import reversal as rv  # noqa: E402

spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
total_it, total_t, losses = 0, 0.0, []
conf = rv.ReversalConfig(tolerance=1e-30, max_iters=iters)
if impl == "gpu-batch":   # every molecule's descent in one batched loop
    grids, peaks = [], []
    for i in range(n_mol + 1):
        ch, xyz = synth.molecule(cfg, i)
        grid, _ = vg.generate_grid(vg.ParticleSet(ch, xyz), spec)
        grids.append(grid)
        peaks.append(rv.detect_peaks(grid, conf.persistence_threshold))
    rv.refine_coords_batch(grids[-1:], peaks[-1:], conf)     # warm-up
    t0 = time.perf_counter()
    states = rv.refine_coords_batch(grids[:n_mol], peaks[:n_mol], conf)
    total_t = time.perf_counter() - t0
    total_it = sum(s_.iterations for s_ in states)
    print(json.dumps({"impl": impl, "workload": f"refine_coords_batch over {n_mol} cfg0 molecules "
                      f"(32^3 x 5) at once, {iters} iterations max each",
                      "iterations": total_it, "seconds": total_t, "iters_per_s": total_it / total_t,
                      "ms_per_iter": total_t / total_it * 1e3,
                      "final_losses": [float(s_.loss) for s_ in states]}))
    sys.exit(0)
for i in [n_mol] + list(range(n_mol)):   # molecule n_mol: untimed warm-up
    warm = i == n_mol
    ch, xyz = synth.molecule(cfg, i)
    grid, _ = vg.generate_grid(vg.ParticleSet(ch, xyz), spec)
    peaks = rv.detect_peaks(grid, conf.persistence_threshold)
    if len(peaks) == 0:
        continue
    t0 = time.perf_counter()
    st = rv.refine_coords(grid, peaks, conf)
    if warm:
        continue
    total_t += time.perf_counter() - t0
    total_it += st.iterations
    losses.append(float(st.loss))
print(json.dumps({"impl": impl, "workload": f"refine_coords on {n_mol} cfg0 molecules "
                  f"(32^3 x 5), {iters} iterations max each", "iterations": total_it,
                  "seconds": total_t, "iters_per_s": total_it / total_t,
                  "ms_per_iter": total_t / total_it * 1e3, "final_losses": losses}))
