"""Wall time of GaussianVoxelizer.transform at cfg1 (1024 molecules as (m, 4)
numpy arrays, D2H of one voxel per grid per call) for several chunk
schedules of loader.generate_rows; prints one JSON line per schedule."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import loader, synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
pb = synth.packed_batch(cfg, range(cfg.n_molecules))
X = [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
     for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
K = 20
for first, cap in ((1 << 20, 1 << 20), (64, 1 << 20), (128, 1 << 20), (256, 1 << 20), (32, 1 << 20),
                   (128, 512), (64, 256)):
    f = lambda: loader.generate_rows(X, spec, first=first, max_chunk=cap)[:, 0, 0, 0, 0].cpu()
    for _ in range(3):
        f()
    ts = []
    for _ in range(K):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ms = float(np.median(ts)) * 1e3
    print(json.dumps({"first": first, "max_chunk": cap, "ms_median": round(ms, 4),
                      "ms_min": round(min(ts) * 1e3, 4),
                      "grids_per_s": round(len(X) / ms * 1e3)}), flush=True)
