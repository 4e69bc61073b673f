"""Step time (default cfg0; args: config batch [variant ...], a variant = "VG_A=1 VG_B=2") (vg_generate_f32, L2 flushed before each step, CUDA events
on the launch stream) for the K13 one-launch path and the K1 + K3 path, per
VG_SMALL_K (float4 slots per thread)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import _native, synth  # noqa: E402

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = synth.CONFIGS[cfgi]
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_molecules
pb = synth.packed_batch(cfg, range(B))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
dev = torch.device("cuda:0")
eng = vg.GridEngine(dev)
lib = _native.lib()
off_d, ch_d, xyz_d = (torch.from_numpy(a).to(dev) for a in (pb.offsets, pb.channels, pb.xyz))
out = torch.empty((B, cfg.channels, *cfg.shape), device=dev)
stats = torch.empty((B, 2), dtype=torch.int64, device=dev)
desc = eng.describe(off_d, ch_d, xyz_d, spec)
lay = _native.VgWsLayout()
lib.vg_workspace_layout(desc, lay)
ws = torch.empty(lay.total, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
scratch = torch.empty(128 << 20, dtype=torch.float32, device=dev)
alg = out.numel() * 4
variants = sys.argv[3:] or ["VG_SMALL=0 VG_PDL=0", "VG_SMALL=0", "VG_SMALL=1"]
for variant in variants:
    for kv in variant.split():
        k, v = kv.split("=")
        os.environ[k] = v
    ts = []
    for it in range(30):
        lib.vg_fill_f32(scratch.data_ptr(), scratch.numel(), 0.0, st)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _native.check(lib.vg_generate_f32(desc, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                          stats.data_ptr(), st), "gen")
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    d = out.view(torch.int32).sum(dim=(1, 2, 3, 4), dtype=torch.int64).cpu().numpy()
    print(json.dumps({"variant": variant, "config": cfgi, "batch": B, "ms": round(ms, 5),
                      "gbs": round(alg / ms / 1e6), "grids_per_s": round(B / ms * 1e3),
                      "digest": int(d.sum() % (1 << 61))}), flush=True)
    for kv in variant.split():
        os.environ.pop(kv.split("=")[0])
