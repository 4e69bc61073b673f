"""Host-side phase times of loader.generate_rows at cfg1 (one call = 1024
molecules): replicates its steps with perf_counter stamps, plus the wait
for the last chunk and the read-back. Median over 20 calls."""
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
pb = synth.packed_batch(cfg, range(cfg.n_molecules))
X = [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
     for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                   cfg.sigma)
pk = _native.pack()
first = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rows = []
for it in range(25):
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    out = torch.empty((1024, 5, 64, 64, 64), device="cuda")
    pipe, lock = loader.shared_pipeline(spec, out.device)
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    pipe.begin(ev)
    T.append(time.perf_counter())
    b = 0
    size = first
    while b < 1024:
        e = min(1024, b + size)
        guess = int((e - b) * pipe.atoms_per_mol * 1.25) + 64
        off, ch, xyz = pipe.staging(e - b, guess)
        T.append(time.perf_counter())
        n = pk.rows_pack(X, b, e, 5, off.ctypes.data, ch.ctypes.data, xyz.ctypes.data, guess)
        T.append(time.perf_counter())
        last = pipe.submit(off, ch[:n], xyz[:n], out=out[b:e], validated=True)
        T.append(time.perf_counter())
        b, size = e, 1 << 30
    cur.wait_event(last.ready)
    v = out[:, 0, 0, 0, 0].cpu()
    T.append(time.perf_counter())
    if it >= 5:
        rows.append(np.diff(T))
r = np.median(np.array(rows), axis=0) * 1e3
names = ["alloc+begin"] + sum([[f"staging{k}", f"pack{k}", f"submit{k}"] for k in range(2)], []) + ["wait+readback"]
print(json.dumps(dict(zip(names, [round(x, 4) for x in r])) | {"total": round(float(r.sum()), 4)}))
