"""CPU baseline: the UNMODIFIED reference package ``voxgrid`` on this host.

Bench infrastructure only (``bench.py``'s ``cpu_baseline`` leg and
``--impl reference``): nothing in the product package imports it. The
reference is installed from /root/reference/pkg into ``baseline/_ref`` by
``scripts/install_reference.sh`` (git-ignored, travels to the GPU box with the
snapshot); on a box without it the callers fall back to the oracle port.

Two figures, as BASELINE.md §3 / SURVEY §8(d) ask, on the SAME molecules the
GPU arm processes (synth.py's seeded BASELINE config batch):

* ``pool``: a process pool of ``ncores`` workers (fork), each calling the
  stock ``voxgrid.generate_grid`` (gridgen.py:130-153) on a contiguous chunk
  of the batch. Workers return the GenStats sums; the grids themselves are
  dropped in the worker (no copy back), which favours the CPU.
* ``generate_batch``: the reference's own parallel API,
  ``voxgrid.generate_batch(sets, spec, parallelism=ncores)``
  (gridgen.py:173-221, ThreadPoolExecutor, GIL-bound).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

REF_DIR = Path(__file__).resolve().parent / "_ref"

_SETS = None    # ParticleSets of the batch (inherited by forked workers)
_SPEC = None


def available() -> bool:
    return (REF_DIR / "voxgrid" / "__init__.py").exists()


def _voxgrid():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import voxgrid

    if not str(Path(voxgrid.__file__).resolve()).startswith(str(REF_DIR.resolve())):
        raise ImportError(f"voxgrid resolved to {voxgrid.__file__}, not baseline/_ref")
    return voxgrid


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def host_info() -> dict:
    """CPU model and numpy's SIMD dispatch (the reference's exp runs there)."""
    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    simd = None
    try:
        from numpy._core import _multiarray_umath as mu

        feats = mu.__cpu_features__
        dispatch = [f for f in mu.__cpu_dispatch__ if feats.get(f)]
        simd = {"baseline": list(mu.__cpu_baseline__), "dispatched": dispatch}
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "numpy": np.__version__, "numpy_simd": simd}


def _build(cfg, pb):
    """Reference ParticleSets + GridSpec for a synth PackedBatch."""
    vx = _voxgrid()
    xyz = pb.xyz.reshape(-1, 3)
    sets = [vx.ParticleSet(pb.channels[a:b].astype(np.int64), xyz[a:b])
            for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
    spec = vx.GridSpec(tuple(cfg.shape), cfg.channels,
                       vx.BoundingBox(tuple(cfg.box_origin), tuple(cfg.box_extents)), cfg.sigma)
    return sets, spec


def _chunk(bounds):
    vx = _voxgrid()
    a, b = bounds
    writes = nonzero = 0
    for i in range(a, b):
        _, st = vx.generate_grid(_SETS[i], _SPEC)
        writes += st.voxel_writes
        nonzero += st.nonzero_voxels
    return writes, nonzero


class RefPool:
    """Process pool over stock ``generate_grid`` for one fixed batch."""

    def __init__(self, cfg, pb, workers: int | None = None):
        global _SETS, _SPEC
        _SETS, _SPEC = _build(cfg, pb)
        self.n = len(_SETS)
        self.workers = workers or host_cores()
        # contiguous chunks, several per worker for balance
        k = max(1, min(self.n, self.workers * 4))
        cuts = np.linspace(0, self.n, k + 1).astype(int)
        self.chunks = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
        self.pool = mp.get_context("fork").Pool(self.workers)

    def run(self):
        """One pass over the batch; returns (voxel_writes, nonzero_voxels) totals."""
        res = self.pool.map(_chunk, self.chunks, chunksize=1)
        return sum(r[0] for r in res), sum(r[1] for r in res)

    def close(self):
        self.pool.close()
        self.pool.join()


def time_pool(cfg, pb, passes: int = 1, warmup: int = 1, workers: int | None = None):
    """grids/s of the process pool over stock generate_grid (full passes)."""
    pool = RefPool(cfg, pb, workers)
    try:
        for _ in range(warmup):
            pool.run()
        t0 = time.perf_counter()
        for _ in range(passes):
            pool.run()
        dt = time.perf_counter() - t0
    finally:
        pool.close()
    return pool.n * passes / dt, dt, pool.workers


def time_generate_batch(cfg, pb, workers: int | None = None):
    """grids/s of the reference's own generate_batch(parallelism=ncores)."""
    vx = _voxgrid()
    sets, spec = _build(cfg, pb)
    workers = workers or host_cores()
    vx.generate_batch(sets[: min(len(sets), 2 * workers)], spec, parallelism=workers)  # warm
    t0 = time.perf_counter()
    res = vx.generate_batch(sets, spec, parallelism=workers)
    dt = time.perf_counter() - t0
    if res.errors:
        raise RuntimeError(f"reference generate_batch failed at {sorted(res.errors)[:4]}")
    return len(sets) / dt, dt, workers
