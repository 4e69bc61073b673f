"""In-process interleaved A/B of K3 variants selected by VG_* hooks (the
library snapshots VG_* at every API call, so one process can switch paths).

python scripts/k3_ab.py CONFIG ROUNDS "label:VG_X=1,VG_Y=2" "label2:VG_X=0" ...

For each variant: K1 once, then per round 10 x (K2 + K3) through
vg_slabs_f32 timed with CUDA events on the launch stream; median over rounds.
Every variant's output must be bit-identical to the first variant's.
"""
import hashlib
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import _native, synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1])]
rounds = int(sys.argv[2])
variants = []
for spec in sys.argv[3:]:
    label, _, envs = spec.partition(":")
    env = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
    variants.append((label, env))
B = min(cfg.n_molecules, 4096)
pb = synth.packed_batch(cfg, range(B))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
dev = torch.device("cuda", 0)
eng = vg.GridEngine(dev)
lib = _native.lib()
off = torch.from_numpy(pb.offsets).to(dev)
ch = torch.from_numpy(pb.channels).to(dev)
xyz = torch.from_numpy(pb.xyz).to(dev)
H, W, D = cfg.shape
out = torch.empty((B, cfg.channels, H, W, D), dtype=torch.float32, device=dev)
stats = torch.empty((B, 2), dtype=torch.int64, device=dev)
desc = eng.describe(off, ch, xyz, spec)
base_env = dict(os.environ)
need = 0
for _, env in variants:   # the bins' size depends on the plan (VG_* hooks)
    os.environ.update(env)
    lay = _native.VgWsLayout()
    _native.check(lib.vg_workspace_layout(desc, lay), "layout")
    need = max(need, lay.total)
    os.environ.clear()
    os.environ.update(base_env)
ws = torch.empty(need, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream(dev)
_native.check(lib.vg_axis_tables_f32(desc, ws.data_ptr(), ws.numel(), st.cuda_stream), "tables")


def run(env, n):
    os.environ.clear()
    os.environ.update(base_env)
    os.environ.update(env)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n):
        _native.check(lib.vg_slabs_f32(desc, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       stats.data_ptr(), st.cuda_stream), "slabs")
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / n


times = {label: [] for label, _ in variants}
digests = {}
for label, env in variants:
    run(env, 3)
    h = hashlib.sha256(out.view(torch.int32).sum(dim=(2, 3, 4)).cpu().numpy().tobytes())
    h.update(out[:, :, ::7, ::5, ::3].contiguous().cpu().numpy().tobytes())
    h.update(stats.cpu().numpy().tobytes())
    digests[label] = h.hexdigest()[:16]
for r in range(rounds):
    for label, env in variants:
        times[label].append(run(env, 10))
alg = B * cfg.grid_bytes
ref = variants[0][0]
for label, _ in variants:
    t = statistics.median(times[label])
    print(f"{cfg.name:24s} {label:28s} K2+K3 {t:.4f} ms  {alg / t / 1e6:7.0f} GB/s  "
          f"range {min(times[label]):.4f}-{max(times[label]):.4f}  digest {digests[label]}"
          f"{'' if digests[label] == digests[ref] else '  MISMATCH'}")
