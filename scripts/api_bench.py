"""Throughput of the reference-facing APIs on the GPU (host packing and
validation included): generate_batch over ParticleSets and
GaussianVoxelizer.transform over (m, 4) arrays, cfg1 (1024 molecules, 64^3 x 5).
python scripts/api_bench.py [reps]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = synth.CONFIGS[1]
pb = synth.packed_batch(cfg, range(cfg.n_molecules))
xyz = pb.xyz.reshape(-1, 3)
sets = [vg.ParticleSet(pb.channels[pb.offsets[b]:pb.offsets[b + 1]].astype(np.int64),
                       xyz[pb.offsets[b]:pb.offsets[b + 1]]) for b in range(pb.n_molecules)]
X = [np.column_stack([s.channels.astype(np.float64), s.positions]) for s in sets]
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
est = vg.GaussianVoxelizer(grid_size=cfg.shape[0], sigma=cfg.sigma, n_channels=cfg.channels,
                           box=(cfg.box_origin, cfg.box_extents)).fit(X)
out = {}
for name, fn in (("generate_batch", lambda: vg.generate_batch(sets, spec).tensor),
                 ("generate_batch per-molecule-bbox",
                  lambda: vg.generate_batch(sets, spec, spec_policy="per-molecule-bbox").tensor),
                 ("GaussianVoxelizer.transform", lambda: est.transform(X))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        t = fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    out[name] = {"ms_per_batch": dt * 1e3, "grids_per_s": pb.n_molecules / dt}
print(json.dumps({"workload": "cfg1: 1024 molecules -> [1024,5,64,64,64] fp32, wall clock "
                  "incl. host validation/packing and H2D", "results": out}))
