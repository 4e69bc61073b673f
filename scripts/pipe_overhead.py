"""Host cost of GridPipeline.submit vs GPU time per batch (cfg0-sized batches)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import synth  # noqa: E402
from paper_2211_08506_b200.loader import GridPipeline  # noqa: E402

cfg = synth.CONFIGS[0]
pb = synth.packed_batch(cfg, range(64))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents), cfg.sigma)
off = torch.as_tensor(pb.offsets).cuda()
ch = torch.as_tensor(pb.channels).cuda()
xyz = torch.as_tensor(pb.xyz).cuda()
pipe = GridPipeline(spec)
for _ in range(20):
    pipe.submit(off, ch, xyz)
pipe.synchronize()
n = 500
t0 = time.perf_counter()
for _ in range(n):
    pipe.submit(off, ch, xyz)
t1 = time.perf_counter()
pipe.synchronize()
t2 = time.perf_counter()
print(f"host submit {(t1 - t0) / n * 1e6:.1f} us/batch; wall {(t2 - t0) / n * 1e6:.1f} us/batch")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    pipe.submit(off, ch, xyz)
pr.disable()
pipe.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
