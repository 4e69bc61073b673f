"""GaussianVoxelizer.transform-style calls at cfg1 (loader.generate_rows, 1024
molecules as (m, 4) arrays) per chunk schedule, in the two consumption modes
of bench.py's e2e_transform: blocking read-back per call, and read-back
queued into pinned memory (sync once at the end). Wall ms per call."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import loader, synth  # noqa: E402

cfg = synth.CONFIGS[1]
pb = synth.packed_batch(cfg, range(cfg.n_molecules))
X = [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
     for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
K = 20
heads = torch.empty((K, 1024), dtype=torch.float32).pin_memory()
for first in (1024, 512, 256, 128, 64):
    f = lambda: loader.generate_rows(X, spec, first=first, max_chunk=8192)
    for _ in range(3):
        f()[:, 0, 0, 0, 0].cpu()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        f()[:, 0, 0, 0, 0].cpu()
    blocking = (time.perf_counter() - t0) / K * 1e3
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        heads[k].copy_(f()[:, 0, 0, 0, 0], non_blocking=True)
    torch.cuda.synchronize()
    queued = (time.perf_counter() - t0) / K * 1e3
    print(json.dumps({"first": first, "blocking_ms": round(blocking, 4),
                      "queued_ms": round(queued, 4)}), flush=True)
