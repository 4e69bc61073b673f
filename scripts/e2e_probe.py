"""Where the e2e step loses time vs the device-resident pipeline (cfg1)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import synth  # noqa: E402
from paper_2211_08506_b200.loader import GridPipeline, pinned_csr  # noqa: E402

cfg = synth.CONFIGS[1]
pb = synth.packed_batch(cfg, range(1024))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents), cfg.sigma)
pipe = GridPipeline(spec)
off_h, ch_h, xyz_h = pinned_csr(pb.offsets, pb.channels, pb.xyz)
off_d, ch_d, xyz_d = off_h.cuda(), ch_h.cuda(), xyz_h.cuda()
st_h = torch.empty((1024, 2), dtype=torch.int64).pin_memory()


def run(name, step, K=20):
    for _ in range(4):
        step()
    pipe.synchronize()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(pipe.compute_stream)
    pipe.begin(a)
    w = time.perf_counter()
    for _ in range(K):
        step()
    b.record(pipe.join())
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    print(f"{name:40s} {ms:.4f} ms/step  wall {(time.perf_counter() - w) / K * 1e3:.4f}")


def dev():
    pipe.submit(off_d, ch_d, xyz_d)


def host_nostats():
    pipe.submit(off_h, ch_h, xyz_h)


def host_stats():
    r = pipe.submit(off_h, ch_h, xyz_h)
    with torch.cuda.stream(pipe.compute_stream):
        st_h.copy_(r.stats, non_blocking=True)


def dev_stats():
    r = pipe.submit(off_d, ch_d, xyz_d)
    with torch.cuda.stream(pipe.compute_stream):
        st_h.copy_(r.stats, non_blocking=True)


for name, f in (("device inputs", dev), ("device inputs + stats D2H", dev_stats),
                ("host inputs", host_nostats), ("host inputs + stats D2H", host_stats)):
    run(name, f)
