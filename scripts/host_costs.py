"""Host cost of each step of one generate_rows call (cfg1 shapes), each
timed in isolation over many repetitions on the GPU box."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import _native, loader, synth  # noqa: E402

cfg = synth.CONFIGS[1]
pb = synth.packed_batch(cfg, range(256))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
res = {}


def t(name, f, n=200):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    res[name] = round((time.perf_counter() - t0) / n * 1e6, 2)
    torch.cuda.synchronize()


keep = []
t("empty_5GB", lambda: keep.append(torch.empty((1024, 5, 64, 64, 64), device="cuda")) or keep.pop(0) if len(keep) > 1 else None)
t("shared_pipeline", lambda: loader.shared_pipeline(spec, "cuda:0"))
dev = torch.device("cuda:0")
t("shared_pipeline_dev", lambda: loader.shared_pipeline(spec, dev))
t("require_cuda", lambda: vg.gridgen._require_cuda(dev))
t("hash_spec", lambda: hash(spec))
pipe, _ = loader.shared_pipeline(spec, dev)
cur = torch.cuda.current_stream()
t("current_stream", lambda: torch.cuda.current_stream(dev))
t("event_record_wait", lambda: (pipe.start_event.record(cur), pipe.copy_stream.wait_event(pipe.start_event)))
t("staging", lambda: pipe.staging(256, 6000), n=50)
out = torch.empty((256, 5, 64, 64, 64), device="cuda")
off, ch, xyz = pipe.staging(256, len(pb.channels))
off[:] = pb.offsets
ch[:] = pb.channels
xyz[:] = pb.xyz.reshape(-1, 3)
t("out_slice", lambda: out[0:256])


def sub():
    pipe.staging(256, len(pb.channels))
    pipe.submit(off, ch, xyz, out=out, validated=True)


t("staging+submit (256 mols)", sub, n=30)
slot = pipe.slots[0]
L = pipe.lib
args = (slot.desc, slot.args, *slot.ptrs)
t("native vg_submit_f32", lambda: L.vg_submit_f32(*args), n=30)
t("native vg_abi_version", lambda: L.vg_abi_version())
print(json.dumps(res))
