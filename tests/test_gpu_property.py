"""Randomised parity (hypothesis, 1000 + 300 derandomised cases): random shapes, channel counts, boxes,
sigmas, thresholds, periodic cells and molecule sizes, GPU path vs the CPU
oracle, bit for bit, with identical GenStats counters. Complements the fixed
cases of test_gpu_parity.py with inputs nobody chose by hand."""

from __future__ import annotations

import numpy as np
import pytest

from _golden import assert_bitwise
from oracle import voxgrid_oracle as orc

torch = pytest.importorskip("torch")
hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

import paper_2211_08506_b200 as vg  # noqa: E402


@st.composite
def batches(draw):
    H = draw(st.integers(1, 40))
    W = draw(st.integers(1, 40))
    D = draw(st.integers(1, 40))
    C = draw(st.integers(1, 6))
    ext = tuple(draw(st.floats(1.0, 12.0)) for _ in range(3))
    origin = tuple(draw(st.floats(-3.0, 3.0)) for _ in range(3))
    periodic = draw(st.booleans())
    max_sigma = min(ext) / 6.0 * 0.99 if periodic else 1.2
    sigma = draw(st.floats(0.05, max(0.05, min(1.2, max_sigma))))
    thr = draw(st.one_of(st.none(), st.floats(1e-7, 0.2)))
    sizes = draw(st.lists(st.integers(0, 40), min_size=1, max_size=6))
    seed = draw(st.integers(0, 2**31 - 1))
    return H, W, D, C, ext, origin, periodic, sigma, thr, sizes, seed


@settings(max_examples=1000, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(batches())
def test_random_batches_match_oracle(case):
    H, W, D, C, ext, origin, periodic, sigma, thr, sizes, seed = case
    if periodic:
        origin = (0.0, 0.0, 0.0)
    rng = np.random.default_rng(seed)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offsets[-1])
    lo = np.array(origin) - 1.5
    hi = np.array(origin) + np.array(ext) + 1.5
    xyz = rng.uniform(lo, hi, (n, 3))
    if periodic:
        xyz = np.mod(xyz, np.array(ext))
    ch = rng.integers(0, C, n).astype(np.int32)
    lattice = vg.LatticeCell(ext) if periodic else None
    spec = vg.GridSpec((H, W, D), C, vg.BoundingBox(origin, ext), sigma, lattice)
    grids, st_ = vg.generate_packed(offsets, ch, xyz, spec, threshold=thr)
    geom = orc.Geometry((H, W, D), C, origin, ext, sigma, periodic)
    ref, rs = orc.batch(offsets, ch, xyz, geom, threshold=thr)
    assert_bitwise(grids.cpu().numpy(), ref, f"random case {case}")
    st_h = st_.cpu().numpy()
    assert [int(v) for v in st_h[:, 0]] == [r["voxel_writes"] for r in rs]
    assert [int(v) for v in st_h[:, 1]] == [r["nonzero_voxels"] for r in rs]


@settings(max_examples=300, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(1, 36), st.integers(1, 36), st.integers(1, 36), st.integers(1, 4),
       st.floats(0.1, 0.9), st.floats(0.0, 6.0),
       st.lists(st.integers(0, 30), min_size=1, max_size=5), st.integers(0, 2**31 - 1))
def test_random_per_molecule_boxes_match_oracle(H, W, D, C, sigma, pad, sizes, seed):
    """spec_policy="per-molecule-bbox" (per-molecule origin and voxel size on
    the device) against the oracle's grids in each molecule's own box."""
    rng = np.random.default_rng(seed)
    sets = [vg.ParticleSet(rng.integers(0, C, n), rng.normal(0.0, 3.0, (n, 3))) for n in sizes]
    spec = vg.GridSpec((H, W, D), C, vg.BoundingBox((0, 0, 0), (1, 1, 1)), sigma)
    res = vg.generate_batch(sets, spec, spec_policy="per-molecule-bbox", padding_sigmas=pad)
    got = res.tensor.cpu().numpy()
    for b, ps in enumerate(sets):
        try:
            origin, ext = orc.bbox_of(np.asarray(ps.positions), sigma, pad)
        except ValueError:
            assert b in res.errors
            assert not got[b].any()
            continue
        assert b not in res.errors
        ref, rs = orc.grid(np.asarray(ps.channels), np.asarray(ps.positions),
                           orc.Geometry((H, W, D), C, origin, ext, sigma))
        assert_bitwise(got[b], ref, f"bbox case {b}")
        g, gs = res.results[b]
        assert gs.voxel_writes == rs["voxel_writes"] and gs.nonzero_voxels == rs["nonzero_voxels"]
