"""Per-axis numerics on the GPU — counterparts of reference ``voxgrid.kernels``.

* ``erf_approx(t)``: the Bürmann-series erf (reference kernels.py:49-70),
  evaluated by the device code in csrc/vg_math.cuh (float32 only).
* ``axis_tables_batch(...)``: every atom's three 1D mass tables and supports
  for a CSR batch (reference fused_axis_tables, kernels.py:217-274) — the
  K1 kernel exposed as an API for consumers such as grid reversal.
* ``fused_axis_tables(mus, axis_params, sigma, ...)``: single-atom form with
  the reference signature, returning ``AxisTable`` objects.
"""

from __future__ import annotations

import numpy as np

from . import _native

__all__ = ["ERF_C1", "ERF_C2", "AxisTable", "erf_approx", "axis_tables_batch",
           "fused_axis_tables"]

ERF_C1 = 31 / 200
ERF_C2 = 341 / 8000


class AxisTable:
    """1D voxel masses of one particle along one axis (kernels.py:101-119);
    all entries outside the half-open ``support`` are exactly zero."""

    __slots__ = ("values", "support")

    def __init__(self, values, support):
        self.values = values
        self.support = (int(support[0]), int(support[1]))

    @property
    def width(self) -> int:
        lo, hi = self.support
        return hi - lo

    def sum(self) -> float:
        return float(np.asarray(self.values, dtype=np.float64).sum())


def _torch():
    import torch

    return torch


def erf_approx(t, dtype=None, device=None):
    """Bürmann erf in float32 on the GPU. Torch CUDA tensors stay on the
    device; numpy arrays / scalars are copied over and back."""
    torch = _torch()
    if dtype is not None and np.dtype(dtype) != np.dtype(np.float32):
        raise ValueError("the GPU erf is float32 only")
    from .gridgen import _require_cuda

    dev = _require_cuda(device)
    as_tensor = isinstance(t, torch.Tensor)
    if as_tensor:
        x = t.to(device=t.device if t.is_cuda else dev, dtype=torch.float32).contiguous()
    else:
        arr = np.asarray(t, dtype=np.float32)
        x = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).to(dev)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    _native.check(_native.lib().vg_erf_f32(x.data_ptr(), out.data_ptr(), x.numel(), stream),
                  "vg_erf_f32")
    if as_tensor:
        return out
    res = out.cpu().numpy().reshape(np.shape(t))
    return float(res) if np.ndim(t) == 0 else res


def axis_tables_batch(offsets, channels, xyz, spec, *, mol_origin=None, mol_delta=None,
                      threshold=None, device=None, engine=None):
    """K1 for a whole CSR batch. Returns device tensors ``(tx (n, W), ty (n, H),
    tz (n, D), supports (n, 3, 2) int32)`` in world axis order x, y, z."""
    torch = _torch()
    from .gridgen import _as_device, default_engine

    eng = engine if engine is not None else default_engine(device)
    dev = eng.device
    off = _as_device(offsets, torch.int64, dev)
    ch = _as_device(channels, torch.int32, dev)
    pos = _as_device(xyz, torch.float64, dev).reshape(-1, 3)
    mo = _as_device(mol_origin, torch.float64, dev) if mol_origin is not None else None
    md = _as_device(mol_delta, torch.float64, dev) if mol_delta is not None else None
    desc = eng.describe(off, ch, pos, spec, mol_origin=mo, mol_delta=md, mode="sparse",
                        threshold=threshold)
    layout = _native.VgWsLayout()
    _native.check(eng.lib.vg_workspace_layout(desc, layout), "vg_workspace_layout")
    ws = torch.empty(layout.total, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(eng.lib.vg_axis_tables_f32(desc, ws.data_ptr(), ws.numel(), stream),
                  "vg_axis_tables_f32")
    n = ch.numel()
    H, W, D = spec.shape

    def view(off_bytes, row, cols):
        t = ws[off_bytes:off_bytes + n * row * 4].view(torch.float32).view(n, row)
        return t[:, :cols]

    tx = view(layout.tx, layout.row_x, W)
    ty = view(layout.ty, layout.row_y, H)
    tz = view(layout.tz, layout.row_z, D)
    sp = ws[layout.supp:layout.supp + n * 16].view(torch.int32).view(n, 4)
    lo = (sp[:, :3] & 0xFFFF)
    hi = (sp[:, :3] >> 16) & 0xFFFF
    supports = torch.stack([lo, hi], dim=2)
    return tx, ty, tz, supports


def fused_axis_tables(mus, axis_params, sigma, dtype=np.float32, threshold=None,
                      periodic=False, device=None):
    """All three axis tables of one particle (reference kernels.py:217-274
    signature); ``axis_params`` is ((n, origin, delta) for x, y, z)."""
    from .core import BoundingBox, GridSpec, LatticeCell

    if np.dtype(dtype) != np.dtype(np.float32):
        raise ValueError("the GPU tables are float32 only")
    (nx, ox, dx), (ny, oy, dy), (nz, oz, dz) = axis_params
    for n, _, d in axis_params:
        if not d > 0.0:
            raise ValueError(f"voxel size must be positive, got {d}")
        if n < 1:
            raise ValueError(f"voxel count must be >= 1, got {n}")
    if not sigma > 0.0:
        raise ValueError(f"sigma must be positive, got {sigma}")
    if periodic:
        for n, _, d in axis_params:
            if not sigma < n * d / 6.0:
                raise ValueError(f"sigma={sigma} too large for periodic cell edge {n * d}; "
                                 "(need sigma < edge/6)")
    ext = (nx * dx, ny * dy, nz * dz)
    spec = GridSpec((ny, nx, nz), 1, BoundingBox((ox, oy, oz), ext), sigma,
                    LatticeCell(ext) if periodic else None)
    # exact per-axis deltas (n*delta/n may differ from delta by an ulp)
    delta = np.array([[dx, dy, dz]], dtype=np.float64)
    origin = np.array([[ox, oy, oz]], dtype=np.float64)
    tx, ty, tz, sup = axis_tables_batch(np.array([0, 1]), np.zeros(1, np.int32),
                                        np.asarray(mus, dtype=np.float64).reshape(1, 3), spec,
                                        mol_origin=origin, mol_delta=delta, threshold=threshold,
                                        device=device)
    sup = sup.cpu().numpy()[0]
    return [AxisTable(t[0].cpu().numpy(), sup[a]) for a, t in enumerate((tx, ty, tz))]
