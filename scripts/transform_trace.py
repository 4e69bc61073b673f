"""Device timeline (torch.profiler / CUPTI) of one GaussianVoxelizer.transform
call at cfg1 with a D2H read-back: every kernel and copy with its start and
end relative to the call, to find the gaps between chunks."""
import sys
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import loader, synth  # noqa: E402

cfg = synth.CONFIGS[1]
pb = synth.packed_batch(cfg, range(cfg.n_molecules))
X = [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
     for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
sched = [(int(a), int(b)) for a, b in (s.split("/") for s in sys.argv[1:])] or [(128, 512)]
for first, cap in sched:
    for _ in range(5):
        loader.generate_rows(X, spec, first=first, max_chunk=cap)[:, 0, 0, 0, 0].cpu()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        loader.generate_rows(X, spec, first=first, max_chunk=cap)[:, 0, 0, 0, 0].cpu()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    cpu = [e for e in prof.events() if e.device_type != torch.autograd.DeviceType.CUDA]
    t0 = min(e.time_range.start for e in cpu)
    print(f"== first={first} max_chunk={cap}")
    for e in sorted(evs, key=lambda e: e.time_range.start):
        print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} "
              f"{e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")
    end = max(e.time_range.end for e in cpu)
    print(f"call end (host) {end - t0:.1f} us")
