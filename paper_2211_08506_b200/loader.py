"""Pipelined batch generation for data loaders.

``GridPipeline`` turns a stream of CSR batches (host or device) into device
grid tensors, overlapping the three stages of consecutive batches on
separate CUDA streams:

    copy stream     H2D of batch k+1's atoms (pinned host -> device)
    tables stream   K1 (per-atom axis tables) of batch k+1
    compute stream  K3 (slab gather/store) of batch k   <- HBM-bound

K1 is compute-bound and K3 HBM-bound, so running them concurrently hides
K1 and the copies behind the grid writes. Inputs, table workspaces and
outputs are double-buffered; every reuse waits on the event of the stage
that last read the buffer, so results are identical to the serial path
(bit for bit: same kernels, same inputs).

The caller consumes ``result.grids`` on ``pipeline.compute_stream`` (or
after ``result.ready.synchronize()``); a slot is rewritten two submissions
later, after the caller's ``release`` event (optional) and the previous
consumer-visible event.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .core import GridSpec
from .gridgen import GridEngine, _require_cuda

__all__ = ["GridPipeline", "PipelineResult"]


@dataclass
class PipelineResult:
    grids: object        # torch.float32 CUDA (B, C, H, W, D); valid after `ready`
    stats: object        # torch.int64 CUDA (B, 2): voxel_writes, nonzero_voxels
    ready: object        # torch.cuda.Event recorded on the compute stream
    slot: int


class _Slot:
    def __init__(self):
        self.off = self.ch = self.xyz = None      # device inputs
        self.ws = None                            # K1 -> K3 tables
        self.out = None
        self.stats = None
        self.done = None                          # K3 finished (inputs/ws/out reusable)
        self.released = None                      # consumer's event (optional)


class GridPipeline:
    """Double-buffered, three-stream generator of grid batches on one device."""

    def __init__(self, spec: GridSpec, device=None, mode: str = "sparse", threshold=None,
                 depth: int = 2):
        import torch

        self.torch = torch
        self.device = _require_cuda(device)
        self.spec = spec
        self.mode = mode
        self.threshold = threshold
        self.engine = GridEngine(self.device)
        self.lib = _native.lib()
        with torch.cuda.device(self.device):
            # K1 (short, compute-bound) runs at high priority so its blocks are
            # dispatched as soon as K3 blocks of the previous batch retire,
            # instead of queueing behind K3's whole grid
            self.copy_stream = torch.cuda.Stream(self.device)
            self.tables_stream = torch.cuda.Stream(self.device, priority=-1)
            self.compute_stream = torch.cuda.Stream(self.device)
        self.slots = [_Slot() for _ in range(depth)]
        self.k = 0
        self.launches = 0

    # -- buffers ---------------------------------------------------------------
    def _ensure(self, t, n, dtype, shape=None):
        torch = self.torch
        need = n if shape is None else int(np.prod(shape))
        if t is None or t.numel() < need or t.dtype != dtype:
            t = torch.empty(max(need, 1), dtype=dtype, device=self.device)
        return t

    def submit(self, offsets, channels, xyz, release=None) -> PipelineResult:
        """Queue one CSR batch (numpy/torch, host or device). Returns at once."""
        torch = self.torch
        spec = self.spec
        slot = self.slots[self.k % len(self.slots)]
        self.k += 1
        B = int(len(offsets) - 1)
        n = int(len(channels))
        H, W, D = spec.shape
        cs, ts, ks = self.copy_stream, self.tables_stream, self.compute_stream

        # the slot's previous K3 must be done before its buffers are rewritten
        for st in (cs, ts, ks):
            if slot.done is not None:
                st.wait_event(slot.done)
            if release is not None:
                st.wait_event(release)
        if _on_device(offsets, torch.int64, self.device) and _on_device(
                channels, torch.int32, self.device) and _on_device(xyz, torch.float64, self.device):
            # device-resident inputs: used in place (caller keeps them unchanged until `ready`)
            off_d, ch_d, xyz_d = offsets, channels, xyz.reshape(-1)
            copied = None
        else:
            slot.off = self._ensure(slot.off, B + 1, torch.int64)
            slot.ch = self._ensure(slot.ch, n, torch.int32)
            slot.xyz = self._ensure(slot.xyz, 3 * n, torch.float64)
            with torch.cuda.stream(cs):
                slot.off[:B + 1].copy_(torch.as_tensor(offsets), non_blocking=True)
                if n:
                    slot.ch[:n].copy_(torch.as_tensor(channels), non_blocking=True)
                    slot.xyz[:3 * n].copy_(torch.as_tensor(xyz).reshape(-1), non_blocking=True)
                copied = torch.cuda.Event()
                copied.record(cs)
            off_d, ch_d, xyz_d = slot.off[:B + 1], slot.ch[:n], slot.xyz[:3 * n]

        desc = self.engine.describe(off_d, ch_d, xyz_d.view(-1, 3), spec, mode=self.mode,
                                    threshold=self.threshold)
        layout = _native.VgWsLayout()
        _native.check(self.lib.vg_workspace_layout(desc, layout), "vg_workspace_layout")
        if slot.ws is None or slot.ws.numel() < layout.total:
            slot.ws = torch.empty(max(layout.total, 1 << 20), dtype=torch.uint8,
                                  device=self.device)
        shape = (B, spec.channels, H, W, D)
        if slot.out is None or tuple(slot.out.shape) != shape:
            slot.out = torch.empty(shape, dtype=torch.float32, device=self.device)
            slot.stats = torch.empty((B, 2), dtype=torch.int64, device=self.device)

        # K1 on the tables stream (after the copy)
        if copied is not None:
            ts.wait_event(copied)
        _native.check(self.lib.vg_axis_tables_f32(desc, slot.ws.data_ptr(), slot.ws.numel(),
                                                  ts.cuda_stream), "vg_axis_tables_f32")
        tabled = torch.cuda.Event()
        tabled.record(ts)
        # K3 on the compute stream (after K1)
        ks.wait_event(tabled)
        _native.check(self.lib.vg_slabs_f32(desc, slot.out.data_ptr(), slot.ws.data_ptr(),
                                            slot.ws.numel(), slot.stats.data_ptr(),
                                            ks.cuda_stream), "vg_slabs_f32")
        done = torch.cuda.Event()
        done.record(ks)
        slot.done = done
        if B:
            self.launches += 2 if n else 1
        # keep the input tensors alive until the copy has happened
        slot._host = (offsets, channels, xyz)
        return PipelineResult(slot.out, slot.stats, done, (self.k - 1) % len(self.slots))

    def begin(self, event):
        """Make every stage wait for ``event`` (e.g. the start of a timed region)."""
        for st in (self.copy_stream, self.tables_stream, self.compute_stream):
            st.wait_event(event)

    def synchronize(self):
        for st in (self.copy_stream, self.tables_stream, self.compute_stream):
            st.synchronize()


def _on_device(t, dtype, device) -> bool:
    import torch

    return (isinstance(t, torch.Tensor) and t.is_cuda and t.device == device and t.dtype == dtype
            and t.is_contiguous())


def pinned_csr(offsets, channels, xyz):
    """Pinned host copies of a CSR batch (fast, asynchronous H2D)."""
    import torch

    return (torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).pin_memory(),
            torch.from_numpy(np.ascontiguousarray(channels, dtype=np.int32)).pin_memory(),
            torch.from_numpy(np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1)).pin_memory())
