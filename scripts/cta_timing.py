"""Per-CTA phase timestamps of K3 (experiment build -DVG_EXP_TIMING, loaded via VG_LIB):
python scripts/cta_timing.py <config> <out.npy>"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import _native, synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1])]
pb = synth.packed_batch(cfg, range(cfg.n_molecules if cfg.n_molecules <= 1024 else 1024))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents), cfg.sigma)
off = torch.as_tensor(pb.offsets).cuda()
ch = torch.as_tensor(pb.channels).cuda()
xyz = torch.as_tensor(pb.xyz).cuda()
for _ in range(4):
    g, st = vg.generate_packed(off, ch, xyz, spec)
torch.cuda.synchronize()
buf = np.zeros((1 << 17, 12), np.uint64)
lib = _native.lib()
fn = lib.vg_exp_timing_fetch
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert fn(buf.ctypes.data, buf.nbytes) == 0
np.save(sys.argv[2], buf)
wbuf = np.zeros((1 << 17, 8), np.uint64)
fw = lib.vg_exp_timing_fetch_warps
fw.restype = ctypes.c_int
fw.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert fw(wbuf.ctypes.data, wbuf.nbytes) == 0
np.save(sys.argv[2].replace(".npy", "_warps.npy"), wbuf)
print("saved", sys.argv[2])
