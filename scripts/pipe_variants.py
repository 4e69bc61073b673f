import sys, time
sys.path.insert(0, '.')
import torch
import paper_2211_08506_b200 as vg
from paper_2211_08506_b200 import synth
from paper_2211_08506_b200.loader import GridPipeline, pinned_csr
cfg = synth.CONFIGS[1]
pb = synth.packed_batch(cfg, range(1024))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents), cfg.sigma)
host = pinned_csr(pb.offsets, pb.channels, pb.xyz)
dev = tuple(t.cuda() for t in host)
st_h = torch.empty((1024, 2), dtype=torch.int64).pin_memory()
for name, inp, so in (("device", dev, None), ("host", host, None), ("host+stats", host, st_h), ("device", dev, None), ("host+stats", host, st_h)):
    pipe = GridPipeline(spec)
    for _ in range(5):
        pipe.submit(*inp, stats_out=so)
    pipe.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(pipe.compute_stream); pipe.begin(a)
    for _ in range(20):
        pipe.submit(*inp, stats_out=so)
    b.record(pipe.join())
    torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 20, 4), "ms/step")
