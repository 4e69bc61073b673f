"""Host cost of one vg_submit_f32 call (tiny batches so the GPU is not the
bound): python scripts/submit_overhead.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import synth  # noqa: E402
from paper_2211_08506_b200.loader import GridPipeline, pinned_csr  # noqa: E402

cfg = synth.CONFIGS[0]
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents), cfg.sigma)
for nmol in (1, 8, 64):
    pb = synth.packed_batch(cfg, range(nmol))
    host = pinned_csr(pb.offsets, pb.channels, pb.xyz)
    dev = tuple(t.cuda() for t in host)
    for name, inputs in (("device", dev), ("pinned host", host)):
        pipe = GridPipeline(spec, depth=4)
        for _ in range(50):
            pipe.submit(*inputs)
        pipe.synchronize()
        n = 2000
        t_call = 0.0
        t0 = time.perf_counter()
        for _ in range(n):
            a = time.perf_counter()
            pipe.submit(*inputs)
            t_call += time.perf_counter() - a
        pipe.synchronize()
        wall = time.perf_counter() - t0
        print(f"{nmol:3d} molecules, {name:11s}: submit {t_call / n * 1e6:6.1f} us/call, "
              f"wall {wall / n * 1e6:6.1f} us/batch")

# the native call alone (descriptor and arguments prepared once)
pb = synth.packed_batch(cfg, range(8))
dev = tuple(torch.from_numpy(a).cuda() for a in (pb.offsets, pb.channels, pb.xyz))
pipe = GridPipeline(spec, depth=1)
pipe.submit(*dev)
pipe.synchronize()
slot = pipe.slots[0]
lib = pipe.lib
args = (slot.desc, slot.args, slot.out.data_ptr(), slot.ws.data_ptr(), slot.ws.numel(),
        slot.stats.data_ptr())
fn = lib.vg_submit_f32
for _ in range(100):
    fn(*args)
torch.cuda.synchronize()
n = 5000
t0 = time.perf_counter()
for _ in range(n):
    fn(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"native vg_submit_f32 alone: {(t1 - t0) / n * 1e6:.1f} us/call")
