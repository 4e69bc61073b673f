"""Write ceiling probes: vg_fill_f32 over the cfg1 output size (5.37 GB) and
torch's fill_, CUDA events, median of 10."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2211_08506_b200 import _native  # noqa: E402

lib = _native.lib()
out = torch.empty(1024 * 5 * 64 ** 3, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for name, f in (("vg_fill_f32", lambda: lib.vg_fill_f32(out.data_ptr(), out.numel(), 0.0, st)),
                ("torch.fill_", lambda: out.fill_(0.0)),
                ("torch.zero_", lambda: out.zero_())):
    ts = []
    for it in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    print(f"{name:16s} {ms:.4f} ms  {out.numel() * 4 / ms / 1e6:.0f} GB/s")
