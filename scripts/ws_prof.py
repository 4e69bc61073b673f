"""K3W wait profile (experiment build -DVG_EXP_WSPROF, loaded with VG_LIB):
python scripts/ws_prof.py CONFIG"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import _native, synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1])]
pb = synth.packed_batch(cfg, range(min(cfg.n_molecules, 1024)))
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents), cfg.sigma)
args = [torch.from_numpy(a).cuda() for a in (pb.offsets, pb.channels, pb.xyz)]
lib = _native.lib()
fn = lib.vg_exp_wsprof
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
for _ in range(2):
    vg.generate_packed(*args, spec, check=False)
torch.cuda.synchronize()
fn(None, 1)
vg.generate_packed(*args, spec, check=False)
torch.cuda.synchronize()
g = np.zeros(8, np.uint64)
fn(g.ctypes.data, 0)
g = g.astype(np.float64)
print(f"consumer warps: waiting for units {g[0] / max(g[1], 1):.3f} of their cycles")
print(f"producer warps: waiting for free slots {g[2] / max(g[3], 1):.3f} of their cycles")
print(f"units {int(g[4])}, candidates staged per unit {g[5] / max(g[4], 1):.1f}")
