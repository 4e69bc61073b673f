"""Grid generation on B200 — drop-in for reference ``voxgrid.gridgen``.

Same entry points, arguments and error behaviour as the reference
(/root/reference/pkg/src/voxgrid/gridgen.py):

* ``generate_grid(points, spec, mode="sparse", dtype=np.float32,
  threshold=None) -> (Grid, GenStats)``                      gridgen.py:130-153
* ``generate_batch(point_sets, spec, spec_policy="fixed", parallelism=1,
  mode="sparse", padding_sigmas=4.0, dtype=np.float32, threshold=None)
  -> BatchResult``                                            gridgen.py:173-221

plus the CSR fast path ``generate_packed`` used by data loaders and the
benchmark. Every grid is computed by the sm_100a kernels behind the C-ABI
(``libvoxgrid_b200.so``); results are bit-identical to the reference's
float32 grids (same erf bits, same fp64 edge arguments, per-voxel
accumulation in input order). Output is device resident:
``BatchResult.tensor`` is one contiguous CUDA tensor ``(B, C, H, W, D)``
and every ``Grid.data`` is a view into it.

``parallelism`` is accepted and validated but does not change anything: the
GPU parallelises across molecules, channels and voxel slabs, and the output
is independent of launch shape (no float atomics), matching the reference's
"parallelism never alters any output" contract (gridgen.py:179-186).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from collections.abc import Sequence

import numpy as np

from . import _native
from .core import BoundingBox, Grid, GridSpec, ParticleSet

__all__ = [
    "GenStats",
    "BatchResult",
    "GridEngine",
    "generate_grid",
    "generate_batch",
    "generate_packed",
    "default_engine",
    "check_packed",
    "flagged_molecules",
]

_MODES = ("dense", "sparse")

# generate_batch runs batches larger than this through the chunked pipeline
# (without an explicit stream / engine); smaller ones in one launch pair
PIPELINE_MIN_BATCH = 128


@dataclass
class GenStats:
    """Work counters of one grid (gridgen.py:39-54)."""

    voxel_writes: int = 0
    erf_evals: int = 0
    nonzero_voxels: int = 0
    elapsed: float = 0.0

    def merge(self, other: "GenStats") -> "GenStats":
        self.voxel_writes += other.voxel_writes
        self.erf_evals += other.erf_evals
        self.elapsed += other.elapsed
        return self


def _check_mode(mode: str) -> None:
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {_MODES}, got {mode!r}")


def _check_dtype(dtype) -> None:
    if np.dtype(dtype) != np.dtype(np.float32):
        raise ValueError(f"the B200 path generates float32 grids only, got {np.dtype(dtype)} "
                         "(float64 grids exist in the reference for gradient tests only)")


def _torch():
    import torch

    return torch


def _require_cuda(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("voxgrid-b200 needs a CUDA device (B200, sm_100a); there is no CPU "
                           "fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


class GridEngine:
    """Per-device launcher: owns the reusable workspace and stats buffers and
    calls ``vg_generate_f32`` on the caller's current stream."""

    def __init__(self, device=None):
        self.device = _require_cuda(device)
        self.lib = _native.lib()
        self._ws = None

    def _workspace(self, nbytes: int):
        torch = _torch()
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self._ws

    def describe(self, offsets, channels, xyz, spec: GridSpec, *, mol_origin=None,
                 mol_delta=None, mode="sparse", threshold=None) -> _native.VgBatchDesc:
        """Fill the C descriptor (device tensors already on self.device)."""
        d = self.describe_spec(spec, mode=mode, threshold=threshold)
        d.n_molecules = int(offsets.numel() - 1)
        d.n_atoms = int(channels.numel())
        d.offsets = offsets.data_ptr()
        d.xyz = xyz.data_ptr() if d.n_atoms else None
        d.channel = channels.data_ptr() if d.n_atoms else None
        d.mol_origin = mol_origin.data_ptr() if mol_origin is not None else None
        d.mol_delta = mol_delta.data_ptr() if mol_delta is not None else None
        return d

    @staticmethod
    def describe_spec(spec: GridSpec, *, mode="sparse", threshold=None) -> _native.VgBatchDesc:
        """A descriptor with the geometry of ``spec`` (no batch pointers yet)."""
        d = _native.VgBatchDesc()
        (_, ox, dx), (_, oy, dy), (_, oz, dz) = spec.axis_params()
        d.origin[:] = (ox, oy, oz)
        d.delta[:] = (dx, dy, dz)
        d.scale = 1.0 / (float(spec.sigma) * math.sqrt(2.0))  # kernels.py:235
        thr = threshold if mode == "sparse" else None           # gridgen.py:94
        d.threshold = float(np.float32(thr)) if thr is not None else float("nan")
        d.periodic = 1 if spec.periodic is not None else 0
        d.H, d.W, d.D = spec.shape
        d.C = spec.channels
        return d

    def run(self, desc: _native.VgBatchDesc, out, stats=None, stream=None) -> None:
        """Launch the path for a filled descriptor: K13 alone for a small batch,
        else K1 (tables), K2 (bins, large molecules) and K3 (slabs)."""
        torch = _torch()
        layout = _native.VgWsLayout()
        _native.check(self.lib.vg_workspace_layout(desc, layout), "vg_workspace_layout")
        ws = self._workspace(layout.total)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        if stream is not None:
            ws.record_stream(stream)   # a later, larger workspace frees it after this launch
        rc = self.lib.vg_generate_f32(desc, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                      stats.data_ptr() if stats is not None else None,
                                      st.cuda_stream)
        _native.check(rc, "vg_generate_f32")


_ENGINES: dict = {}


def default_engine(device=None) -> GridEngine:
    dev = _require_cuda(device)
    eng = _ENGINES.get(dev.index)
    if eng is None:
        eng = _ENGINES[dev.index] = GridEngine(dev)
    return eng


def _molecule_of(offsets: np.ndarray, atoms: np.ndarray) -> np.ndarray:
    """Molecule index of each atom index (CSR offsets, empty molecules skipped)."""
    return np.searchsorted(offsets, atoms, side="right") - 1


def check_packed(offsets, channels, xyz, n_channels: int) -> None:
    """Vectorised input validation of a host CSR batch, with the reference's
    rules and exception type: channels in [0, C) (gridgen.py:86-87, 114-119;
    core.py:190-191) and finite positions (gridgen.py:88-90; core.py:197-198).
    Raises ValueError naming the first offending molecule."""
    off = np.asarray(offsets)
    ch = np.asarray(channels)
    if ch.size and not (ch.min() >= 0 and ch.max() < n_channels):
        bad = (ch < 0) | (ch >= n_channels)
        if bad.any():
            a = int(np.flatnonzero(bad)[0])
            b = int(_molecule_of(off, np.array([a]))[0])
            if int(ch[a]) < 0:
                raise ValueError(f"molecule {b}: channel indices must be nonnegative")
            raise ValueError(f"molecule {b}: particle channel {int(ch[a])} out of range for spec "
                             f"with {n_channels} channels")
    pos = np.asarray(xyz)
    if pos.size and not np.isfinite(pos.sum()):   # fast path: a finite sum means all finite
        fin = np.isfinite(pos.reshape(-1, 3)).all(axis=1)
        if not fin.all():
            a = int(np.flatnonzero(~fin)[0])
            b = int(_molecule_of(off, np.array([a]))[0])
            raise ValueError(f"molecule {b}: particle positions must be finite")


def flagged_molecules(stats) -> np.ndarray:
    """Molecules whose kernel stats carry the invalid-atom flag
    (voxel_writes < 0: an atom with a channel outside [0, C) or a non-finite
    position was found on the device and not splatted)."""
    st = stats.cpu().numpy() if hasattr(stats, "cpu") else np.asarray(stats)
    return np.flatnonzero(st[:, 0] < 0) if st.size else np.zeros(0, dtype=np.int64)


def raise_if_flagged(stats) -> None:
    bad = flagged_molecules(stats)
    if bad.size:
        raise ValueError(f"molecules {bad.tolist()[:16]} hold particles with a channel outside "
                         "[0, C) or a non-finite position (reference ValueError, "
                         "gridgen.py:86-90); they were not splatted")


def _is_device(*arrs) -> bool:
    torch = _torch()
    return any(isinstance(a, torch.Tensor) and a.is_cuda for a in arrs)


def _as_device(arr, dtype, device):
    torch = _torch()
    if isinstance(arr, torch.Tensor):
        return arr.to(device=device, dtype=dtype, non_blocking=True).contiguous()
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device=device, dtype=dtype,
                                                          non_blocking=True)


def generate_packed(offsets, channels, xyz, spec: GridSpec, *, mol_origin=None, mol_delta=None,
                    mode: str = "sparse", threshold: float | None = None, out=None,
                    with_stats: bool = True, device=None, stream=None, engine=None,
                    check: bool = True):
    """CSR fast path: molecule b owns atoms ``offsets[b]:offsets[b+1]``.

    ``offsets`` int64 (B+1,), ``channels`` int (n,), ``xyz`` float64 (n, 3),
    numpy arrays or torch tensors (host or device). Optional ``mol_origin`` /
    ``mol_delta`` (B, 3) fp64 give per-molecule boxes (x, y, z order).
    Returns ``(grids, stats)``: grids a CUDA float32 ``(B, C, H, W, D)``
    tensor, stats an int64 ``(B, 2)`` device tensor ``[voxel_writes,
    nonzero_voxels]`` (sparse-mode support volumes) or None.

    Validation follows the reference (ValueError for a channel outside
    [0, C) or a non-finite position, gridgen.py:86-90): host inputs are
    checked on the host before the launch; device-resident inputs are
    checked by K1, which flags the molecule (``voxel_writes < 0``) instead of
    splatting the atom, and with ``check=True`` the flag is read back (one
    synchronisation) and raised. ``check=False`` skips that read-back: test
    ``stats[:, 0] < 0`` yourself (``flagged_molecules``).
    """
    torch = _torch()
    _check_mode(mode)
    eng = engine if engine is not None else default_engine(device)
    dev = eng.device
    on_device = _is_device(offsets, channels, xyz)
    if not on_device:
        check_packed(offsets, channels, xyz, spec.channels)
    offsets_d = _as_device(offsets, torch.int64, dev)
    channels_d = _as_device(channels, torch.int32, dev)
    xyz_d = _as_device(xyz, torch.float64, dev).reshape(-1, 3)
    if channels_d.numel() != xyz_d.shape[0]:
        raise ValueError(f"channel/position count mismatch: {channels_d.numel()} vs "
                         f"{xyz_d.shape[0]}")
    B = offsets_d.numel() - 1
    if B < 0:
        raise ValueError("offsets must hold B+1 >= 1 entries")
    mo = _as_device(mol_origin, torch.float64, dev) if mol_origin is not None else None
    md = _as_device(mol_delta, torch.float64, dev) if mol_delta is not None else None
    H, W, D = spec.shape
    if out is None:
        out = torch.empty((B, spec.channels, H, W, D), dtype=torch.float32, device=dev)
    elif (tuple(out.shape) != (B, spec.channels, H, W, D) or out.dtype != torch.float32
          or not out.is_contiguous() or out.device != dev):
        raise ValueError("out must be a contiguous float32 (B, C, H, W, D) tensor on the device")
    need_flag = on_device and check
    stats = (torch.empty((B, 2), dtype=torch.int64, device=dev)
             if with_stats or need_flag else None)
    desc = eng.describe(offsets_d, channels_d, xyz_d, spec, mol_origin=mo, mol_delta=md,
                        mode=mode, threshold=threshold)
    eng.run(desc, out, stats, stream)
    if need_flag and B:
        if stream is not None:
            stream.synchronize()
        raise_if_flagged(stats)
    return out, (stats if with_stats else None)


@dataclass
class BatchResult:
    """Per-molecule outcomes; failures never abort the batch (gridgen.py:156-170).

    ``tensor`` holds every grid (failed molecules' slots are zero);
    ``results[b]`` is ``(Grid, GenStats)`` or None for failed molecules.
    Stats are copied to the host on first access of ``results``.
    """

    tensor: object
    specs: list
    errors: dict = field(default_factory=dict)
    _stats_dev: object = None
    _atoms: np.ndarray | None = None
    _mode: str = "sparse"
    _images: int = 1
    _elapsed: float = 0.0
    _results: list | None = None

    def __len__(self) -> int:
        return len(self.specs)

    @property
    def results(self) -> list:
        if self._results is None:
            self._results = self._materialize()
        return self._results

    def _materialize(self) -> list:
        B = len(self.specs)
        st = self._stats_dev.cpu().numpy() if (self._stats_dev is not None and B) else None
        per = self._elapsed / B if B else 0.0
        out = []
        for b, spec in enumerate(self.specs):
            if b in self.errors:
                out.append(None)
                continue
            n = int(self._atoms[b])
            H, W, D = spec.shape
            evals = n * self._images * ((W + 1) + (H + 1) + (D + 1))
            writes = int(st[b, 0]) if self._mode == "sparse" else n * H * W * D
            gs = GenStats(voxel_writes=writes, erf_evals=evals,
                          nonzero_voxels=int(st[b, 1]), elapsed=per)
            out.append((Grid(spec, self.tensor[b]), gs))
        return out

    def grids(self) -> list:
        if self.errors:
            bad = sorted(self.errors)
            raise ValueError(f"batch had failures at indices {bad}: {self.errors[bad[0]]}")
        return [g for g, _ in self.results]


def _consistency_error(points, spec: GridSpec):
    """The reference's per-molecule checks (gridgen.py:114-127, kernels.py:239-246)."""
    n = len(points)
    if n and int(np.max(points.channels)) >= spec.channels:
        return ValueError(f"particle channel {int(np.max(points.channels))} out of range "
                          f"for spec with {spec.channels} channels")
    lattice = getattr(points, "lattice", None)
    if (lattice is None) != (spec.periodic is None):
        return ValueError("particle set and spec disagree on periodicity")
    if lattice is not None and spec.periodic is not None:
        if tuple(lattice.edges) != tuple(spec.periodic.edges):
            return ValueError(f"lattice mismatch: points {lattice.edges} vs spec "
                              f"{spec.periodic.edges}")
    if n and spec.periodic is not None:
        for cnt, _, delta in spec.axis_params():
            edge = cnt * delta
            if not spec.sigma < edge / 6.0:
                return ValueError(
                    f"sigma={spec.sigma} too large for periodic cell edge {edge}; wrapped mass "
                    "beyond the nearest images would be lost (need sigma < edge/6)")
    return None


class _BoxSpecs(Sequence):
    """Per-molecule GridSpecs of the per-molecule-bbox policy, built on access
    (a batch of thousands of molecules should not pay for thousands of
    validated GridSpec objects up front)."""

    def __init__(self, spec: GridSpec, origin: np.ndarray, extents: np.ndarray, errors: dict):
        self._spec, self._origin, self._extents, self._errors = spec, origin, extents, errors

    def __len__(self) -> int:
        return len(self._origin)

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self[i] for i in range(*b.indices(len(self)))]
        if b < 0:
            b += len(self)
        if b in self._errors:
            return self._spec
        box = BoundingBox(tuple(self._origin[b].tolist()), tuple(self._extents[b].tolist()))
        s = self._spec
        return GridSpec(s.shape, s.channels, box, s.sigma, s.periodic)


def _bbox_policy(sets, spec: GridSpec, padding_sigmas: float, errors: dict):
    """Per-molecule padded boxes (gridgen.py:192-197 + core.py:283-312), in
    fp64 with the reference's exact op order, vectorised over the batch;
    returns (origin, delta, specs)."""
    B = len(sets)
    origin = np.zeros((B, 3))
    delta = np.ones((B, 3))
    extents = np.ones((B, 3))
    H, W, D = spec.shape
    pad = padding_sigmas * float(spec.sigma)
    counts = np.array([len(ps) for ps in sets], dtype=np.int64)
    live = np.array([b not in errors for b in range(B)], dtype=bool)
    if padding_sigmas < 0.0:
        for b in np.flatnonzero(live):
            errors[int(b)] = ValueError(f"padding_sigmas must be >= 0, got {padding_sigmas}")
        return origin, delta, _BoxSpecs(spec, origin, extents, errors)
    for b in np.flatnonzero(live & (counts == 0)):
        errors[int(b)] = ValueError("cannot compute a bounding box of an empty particle set")
    use = np.flatnonzero(live & (counts > 0))
    if use.size:
        pos = np.concatenate([np.asarray(sets[b].positions, dtype=np.float64) for b in use])
        starts = np.concatenate([[0], np.cumsum(counts[use])[:-1]])
        lo = np.minimum.reduceat(pos, starts, axis=0) - pad
        hi = np.maximum.reduceat(pos, starts, axis=0) + pad
        ext = np.maximum(hi - lo, 0.0)
        org = 0.5 * (lo + hi) - 0.5 * ext
        bad = ext.min(axis=1) <= 0.0
        for b in use[bad]:
            errors[int(b)] = ValueError("degenerate bounding box (zero extent on some axis); "
                                        "use padding_sigmas > 0 or a positive min_extent")
        # overflowing boxes: record whatever GridSpec validation raises, as before
        odd = ~bad & ~(np.isfinite(ext).all(axis=1) & np.isfinite(org).all(axis=1))
        for i in np.flatnonzero(odd):
            try:
                GridSpec(spec.shape, spec.channels,
                         BoundingBox(tuple(org[i].tolist()), tuple(ext[i].tolist())),
                         spec.sigma, spec.periodic)
            except Exception as exc:  # noqa: BLE001 - recorded per index like the reference
                errors[int(use[i])] = exc
                bad[i] = True
        ok = use[~bad]
        origin[ok] = org[~bad]
        extents[ok] = ext[~bad]
        delta[ok] = ext[~bad] / np.array([W, H, D], dtype=np.float64)
    return origin, delta, _BoxSpecs(spec, origin, extents, errors)


def _batch_errors(sets: Sequence, spec: GridSpec) -> dict:
    """Per-index consistency errors (gridgen.py:114-127): vectorised channel
    check; per-molecule checks only where periodicity is involved or a
    molecule fails (for the reference's exact message)."""
    errors: dict = {}
    C = spec.channels
    periodic = spec.periodic is not None
    suspects = [b for b, ps in enumerate(sets)
                if periodic or getattr(ps, "lattice", None) is not None]
    if sets:
        maxch = _max_channels(sets)
        suspects = sorted(set(suspects) | set(np.flatnonzero(maxch >= C).tolist()))
    for b in suspects:
        exc = _consistency_error(sets[b], spec)
        if exc is not None:
            errors[b] = exc
    return errors


def _max_channels(sets: Sequence) -> np.ndarray:
    counts = np.array([len(ps) for ps in sets], dtype=np.int64)
    out = np.full(len(sets), -1, dtype=np.int64)
    nz = np.flatnonzero(counts)
    if nz.size:
        ch = np.concatenate([sets[b].channels for b in nz])
        starts = np.concatenate([[0], np.cumsum(counts[nz])[:-1]])
        out[nz] = np.maximum.reduceat(ch, starts)
    return out


def pack_particle_sets(sets: Sequence, spec: GridSpec, errors: dict):
    """CSR arrays of every molecule without a recorded error (failed molecules
    get an empty atom range, hence an all-zero grid slot)."""
    B = len(sets)
    counts = np.array([len(ps) for ps in sets], dtype=np.int64).reshape(B)
    for b in errors:
        counts[b] = 0
    offsets = np.zeros(B + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    keep = np.flatnonzero(counts)
    if keep.size:
        channels = np.concatenate([sets[b].channels for b in keep]).astype(np.int32)
        xyz = np.concatenate([np.asarray(sets[b].positions, dtype=np.float64).reshape(-1, 3)
                              for b in keep])
    else:
        channels = np.empty(0, dtype=np.int32)
        xyz = np.empty((0, 3), dtype=np.float64)
    return offsets, channels, xyz, counts


def generate_batch(point_sets: Sequence, spec: GridSpec, spec_policy: str = "fixed",
                   parallelism: int = 1, mode: str = "sparse", padding_sigmas: float = 4.0,
                   dtype=np.float32, threshold: float | None = None, *, device=None,
                   stream=None, engine=None) -> BatchResult:
    """One grid per particle set, all in one device tensor (gridgen.py:173-221).

    ``spec_policy="fixed"`` shares ``spec``; ``"per-molecule-bbox"`` keeps
    shape/channels/sigma and fits each molecule its own padded box.
    Per-molecule failures are recorded in ``errors`` and never abort the batch.
    """
    if spec_policy not in ("fixed", "per-molecule-bbox"):
        raise ValueError(f"unknown spec_policy {spec_policy!r}")
    if parallelism < 1:
        raise ValueError(f"parallelism must be >= 1, got {parallelism}")
    _check_mode(mode)
    _check_dtype(dtype)
    start = time.perf_counter()
    errors = _batch_errors(point_sets, spec)
    mol_origin = mol_delta = None
    specs = [spec] * len(point_sets)
    if spec_policy == "per-molecule-bbox":
        mol_origin, mol_delta, specs = _bbox_policy(point_sets, spec, padding_sigmas, errors)
    if stream is None and engine is None and len(point_sets) > PIPELINE_MIN_BATCH:
        # large batch: chunks gathered into pinned staging while the device
        # works on the previous chunk (loader.generate_sets)
        from .loader import generate_sets

        counts = np.array([len(ps) for ps in point_sets], dtype=np.int64).reshape(-1)
        for b in errors:
            counts[b] = 0
        tensor, stats = generate_sets(point_sets, spec, counts, mol_origin=mol_origin,
                                      mol_delta=mol_delta, device=device, mode=mode,
                                      threshold=threshold)
    else:
        offsets, channels, xyz, counts = pack_particle_sets(point_sets, spec, errors)
        tensor, stats = generate_packed(offsets, channels, xyz, spec, mol_origin=mol_origin,
                                        mol_delta=mol_delta, mode=mode, threshold=threshold,
                                        device=device, stream=stream, engine=engine)
    images = 3 if spec.periodic is not None else 1
    return BatchResult(tensor, specs, errors, stats, counts, mode, images,
                       time.perf_counter() - start)


def generate_grid(points, spec: GridSpec, mode: str = "sparse", dtype=np.float32,
                  threshold: float | None = None, *, device=None, stream=None,
                  engine=None):
    """Splat every particle into a fresh device grid (gridgen.py:130-153)."""
    _check_mode(mode)
    _check_dtype(dtype)
    exc = _consistency_error(points, spec)
    if exc is not None:
        raise exc
    res = generate_batch([points], spec, mode=mode, threshold=threshold, device=device,
                         stream=stream, engine=engine)
    grid, stats = res.results[0]
    stats.elapsed = res._elapsed
    return grid, stats
