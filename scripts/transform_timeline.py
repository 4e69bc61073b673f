"""Where the time of a transform call goes (cfg1): host time until
generate_rows returns, device span (events on the caller's stream around the
call), and total until the D2H read-back; per chunk schedule."""
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
cur = torch.cuda.current_stream()
for first, cap in ((1 << 20, 1 << 20), (128, 256), (256, 256), (512, 512), (128, 512)):
    rec = []
    for it in range(23):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(cur)
        g = loader.generate_rows(X, spec, first=first, max_chunk=cap)
        t1 = time.perf_counter()
        e1.record(cur)
        v = g[:, 0, 0, 0, 0].cpu()
        t2 = time.perf_counter()
        if it >= 3:
            rec.append((t1 - t0, e0.elapsed_time(e1) * 1e-3, t2 - t0))
    r = np.median(np.array(rec), axis=0) * 1e3
    print(json.dumps({"first": first, "max_chunk": cap, "host_ms": round(r[0], 4),
                      "device_span_ms": round(r[1], 4), "total_ms": round(r[2], 4)}), flush=True)
# pre-packed, one pipeline submit into a fresh output (the bench's e2e shape)
pipe = loader.GridPipeline(spec)
pin = loader.pinned_csr(pb.offsets, pb.channels, pb.xyz)
rec = []
for it in range(23):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = torch.empty((1024, 5, 64, 64, 64), device="cuda")
    r = pipe.submit(*pin, out=out)
    cur.wait_event(r.ready)
    t1 = time.perf_counter()
    v = out[:, 0, 0, 0, 0].cpu()
    t2 = time.perf_counter()
    if it >= 3:
        rec.append((t1 - t0, t2 - t0))
r = np.median(np.array(rec), axis=0) * 1e3
print(json.dumps({"prepacked_submit_host_ms": round(r[0], 4), "total_ms": round(r[1], 4)}))
