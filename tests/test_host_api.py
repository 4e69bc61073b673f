"""Host-side logic of the drop-in API (no GPU): geometry types, validation
and error behaviour mirrored from the reference (core.py, gridgen.py,
estimator.py, validation.py), CSR packing, per-molecule boxes, and the
no-fallback rule (GPU entry points fail loudly without CUDA)."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2211_08506_b200 as vg
from _golden import config_records
from oracle import voxgrid_oracle as orc
from paper_2211_08506_b200 import gridgen, synth


# --- core types (reference core.py:52-166, test_core.py) ----------------------
def test_bounding_box_and_lattice_validation():
    box = vg.BoundingBox((0, 1, 2), (3, 4, 5))
    assert box.max_corner == (3.0, 5.0, 7.0)
    assert box.translate((1, 1, 1)).origin == (1.0, 2.0, 3.0)
    assert box.contains((1, 2, 3)) and not box.contains((4, 2, 3))
    for bad in [((0, 0, 0), (1, 0, 1)), ((0, 0), (1, 1, 1)), ((0, 0, math.nan), (1, 1, 1))]:
        with pytest.raises(ValueError):
            vg.BoundingBox(*bad)
    with pytest.raises(ValueError):
        vg.LatticeCell((1, -1, 1))


def test_gridspec_validation_and_axis_params():
    box = vg.BoundingBox((-1, 0, 2), (3, 4, 2.5))
    spec = vg.GridSpec((7, 6, 5), 1, box, 0.4)
    assert spec.voxel_sizes == (3 / 6, 4 / 7, 2.5 / 5)
    assert spec.axis_params() == ((6, -1.0, 0.5), (7, 0.0, 4 / 7), (5, 2.0, 0.5))
    assert spec.voxel_count == 7 * 6 * 5
    assert vg.GridSpec.cubic(8, 2, box, 0.3).shape == (8, 8, 8)
    for shape, ch, sigma in [((0, 1, 1), 1, 0.1), ((1, 1), 1, 0.1), ((2, 2, 2), 0, 0.1),
                             ((2, 2, 2), 1, 0.0), ((2, 2, 2), 1, math.inf)]:
        with pytest.raises(ValueError):
            vg.GridSpec(shape, ch, box, sigma)
    with pytest.raises(ValueError):  # periodic cell must equal the box
        vg.GridSpec((4, 4, 4), 1, vg.BoundingBox((0, 0, 0), (6, 6, 6)), 0.3,
                    vg.LatticeCell((6, 6, 7)))


def test_particle_set_semantics():
    ps = vg.ParticleSet([0.0, 2.0], [[1, 2, 3], [4, 5, 6]])
    assert ps.channels.dtype == np.int64 and ps.positions.dtype == np.float64
    assert not ps.channels.flags.writeable and not ps.positions.flags.writeable
    assert len(ps) == 2 and ps.n_channels == 3
    assert list(ps) == [(0, (1.0, 2.0, 3.0)), (2, (4.0, 5.0, 6.0))]
    assert np.array_equal(ps.channel_counts(4), [1, 0, 1, 0])
    assert np.array_equal(vg.ParticleSet.from_rows(ps.to_rows()).positions, ps.positions)
    assert len(vg.ParticleSet.from_rows([])) == 0
    cell = vg.LatticeCell((6.0, 6.0, 6.0))
    wrapped = vg.ParticleSet([0], [[-0.5, 6.5, 3.0]], cell)
    assert np.array_equal(wrapped.positions, np.mod([[-0.5, 6.5, 3.0]], 6.0))
    for ch, pos in [([0.5], [[0, 0, 0]]), ([-1], [[0, 0, 0]]), ([0], [[0, np.nan, 0]]),
                    ([0, 1], [[0, 0, 0]])]:
        with pytest.raises(ValueError):
            vg.ParticleSet(ch, pos)
    with pytest.raises(ValueError):
        vg.ParticleSet.from_rows([[0, 1, 2]])


def test_voxel_world_round_trip():
    spec = vg.GridSpec((4, 5, 6), 1, vg.BoundingBox((-1, 0, 2), (5, 4, 3)), 0.3)
    rng = np.random.default_rng(1)
    for _ in range(50):
        p = [o + rng.uniform(1e-6, e - 1e-6) for o, e in zip(spec.box.origin, spec.box.extents)]
        idx = vg.world_to_voxel(spec, p)
        corner = vg.voxel_to_world(spec, idx)
        for a, (_, _, d) in enumerate(spec.axis_params()):
            assert corner[a] <= p[a] < corner[a] + d
    with pytest.raises(ValueError):
        vg.world_to_voxel(spec, (99, 0, 0))
    with pytest.raises(IndexError):
        vg.voxel_to_world(spec, (9, 0, 0))


def test_bounding_box_of_matches_oracle_and_golden():
    rec = [r for r in config_records()["batches"] if r["spec_policy"] == "per-molecule-bbox"][0]
    cfg = synth.CONFIGS[rec["config"]]
    pb = synth.packed_batch(cfg, rec["indices"])
    for b, g in enumerate(rec["grids"]):
        ch, xyz = pb.molecule(b)
        box = vg.bounding_box_of(vg.ParticleSet(ch, xyz), cfg.sigma, 4.0)
        assert [list(box.origin), list(box.extents)] == g["box"]
        assert (box.origin, box.extents) == orc.bbox_of(xyz, cfg.sigma, 4.0)
    with pytest.raises(ValueError):
        vg.bounding_box_of(vg.ParticleSet.from_rows([]), 0.5)
    with pytest.raises(ValueError):
        vg.bounding_box_of(vg.ParticleSet([0], [[0, 0, 0]]), 0.5, padding_sigmas=0.0)
    floored = vg.bounding_box_of(vg.ParticleSet([0], [[1, 2, 3]]), 0.5, 0.0, min_extent=2.0)
    assert floored.extents == (2.0, 2.0, 2.0) and floored.origin == (0.0, 1.0, 2.0)


# --- batch packing and per-index errors (gridgen.py:114-127, 173-221) ----------
def test_pack_and_consistency_errors():
    spec = vg.GridSpec((8, 8, 8), 2, vg.BoundingBox((0, 0, 0), (4, 4, 4)), 0.3)
    sets = [vg.ParticleSet([0, 1], [[1, 1, 1], [2, 2, 2]]), vg.ParticleSet([5], [[2, 2, 2]]),
            vg.ParticleSet.from_rows([]), vg.ParticleSet([1], [[3, 3, 3]])]
    errors = {}
    for b, ps in enumerate(sets):
        exc = gridgen._consistency_error(ps, spec)
        if exc is not None:
            errors[b] = exc
    assert list(errors) == [1] and "out of range" in str(errors[1])
    offsets, ch, xyz, counts = gridgen.pack_particle_sets(sets, spec, errors)
    assert offsets.tolist() == [0, 2, 2, 2, 3]
    assert ch.tolist() == [0, 1, 1] and counts.tolist() == [2, 0, 0, 1]
    assert np.array_equal(xyz, [[1, 1, 1], [2, 2, 2], [3, 3, 3]])
    cell = vg.LatticeCell((4.0, 4.0, 4.0))
    assert gridgen._consistency_error(vg.ParticleSet([0], [[1, 1, 1]], cell), spec) is not None
    pspec = vg.GridSpec((8, 8, 8), 1, vg.BoundingBox((0, 0, 0), (4, 4, 4)), 0.9, cell)
    assert "too large" in str(gridgen._consistency_error(vg.ParticleSet([0], [[1, 1, 1]], cell),
                                                          pspec))
    assert gridgen._consistency_error(vg.ParticleSet.from_rows([], cell), pspec) is None


def test_bbox_policy_matches_bounding_box_of():
    spec = vg.GridSpec((16, 12, 8), 1, vg.BoundingBox((0, 0, 0), (1, 1, 1)), 0.4)
    sets = [vg.ParticleSet([0], [[100.0, 100.0, 100.0]]), vg.ParticleSet.from_rows([]),
            vg.ParticleSet([0, 0], [[-50.0, 0.0, 0.0], [-49.0, 1.0, 3.0]])]
    errors = {}
    origin, delta, specs = gridgen._bbox_policy(sets, spec, 4.0, errors)
    assert list(errors) == [1]
    for b in (0, 2):
        box = vg.bounding_box_of(sets[b], 0.4, 4.0)
        assert specs[b].box == box
        assert tuple(origin[b]) == box.origin
        assert tuple(delta[b]) == (box.extents[0] / 12, box.extents[1] / 16, box.extents[2] / 8)


def test_argument_validation_without_gpu():
    spec = vg.GridSpec((4, 4, 4), 1, vg.BoundingBox((0, 0, 0), (1, 1, 1)), 0.1)
    with pytest.raises(ValueError):
        vg.generate_batch([], spec, spec_policy="nope")
    with pytest.raises(ValueError):
        vg.generate_batch([], spec, parallelism=0)
    with pytest.raises(ValueError):
        vg.generate_batch([], spec, mode="fast")
    with pytest.raises(ValueError):
        vg.generate_batch([], spec, dtype=np.float64)


def test_gpu_entry_points_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present: covered by the GPU suite")
    spec = vg.GridSpec((4, 4, 4), 1, vg.BoundingBox((0, 0, 0), (1, 1, 1)), 0.1)
    with pytest.raises(RuntimeError, match="no CPU\\s+fallback|CPU fallback"):
        vg.generate_grid(vg.ParticleSet([0], [[0.5, 0.5, 0.5]]), spec)
    with pytest.raises(RuntimeError):
        vg.generate_packed(np.array([0, 1]), np.zeros(1, np.int32), np.zeros((1, 3)), spec)
    with pytest.raises(RuntimeError):
        vg.erf_approx(np.zeros(3, np.float32))


# --- estimator (estimator.py:52-151, test_estimator.py) -----------------------
def sample_clouds():
    return [np.array([[0, 2.0, 2.0, 2.0], [1, 4.0, 3.5, 2.5]]), np.array([[0, 3.0, 4.0, 5.0]])]


def test_estimator_params_clone_and_fit():
    from sklearn.base import clone

    est = vg.GaussianVoxelizer(grid_size=16, sigma=0.3)
    assert est.get_params()["grid_size"] == 16
    est.set_params(sigma=0.7)
    assert clone(est).get_params() == est.get_params()
    est = vg.GaussianVoxelizer(grid_size=16, sigma=0.4).fit(sample_clouds())
    assert est.channels_ == 2
    pad = 4 * 0.4
    assert np.allclose(est.box_.origin, [2 - pad, 2 - pad, 2 - pad])
    assert np.allclose(est.box_.max_corner, [4 + pad, 4 + pad, 5 + pad])
    rec = config_records()["estimator"]["shared"]
    clouds = []
    for b in range(6):
        ch, xyz = synth.molecule(synth.CONFIGS[0], b)
        clouds.append(np.column_stack([ch.astype(np.float64), xyz]))
    est = vg.GaussianVoxelizer(grid_size=24, sigma=0.4).fit(clouds)
    assert [list(est.box_.origin), list(est.box_.extents)] == rec["box"]
    assert est.channels_ == rec["channels"]


def test_estimator_box_modes_and_validation():
    explicit = vg.GaussianVoxelizer(box=((0, 0, 0), (8, 8, 8))).fit(sample_clouds())
    assert explicit.box_.extents == (8, 8, 8)
    assert vg.GaussianVoxelizer(box="per-sample").fit(sample_clouds()).box_ is None
    per = vg.GaussianVoxelizer(periodic=(6, 6, 6)).fit(sample_clouds())
    assert per.box_ == vg.BoundingBox((0, 0, 0), (6, 6, 6))
    with pytest.raises(ValueError):
        vg.GaussianVoxelizer(periodic=(6, 6, 6), box=((0, 0, 0), (6, 6, 6))).fit(sample_clouds())
    with pytest.raises(RuntimeError):
        vg.GaussianVoxelizer().transform(sample_clouds())
    est = vg.GaussianVoxelizer(grid_size=8, sigma=0.3)
    for bad in ([np.array([[0, 1, 2]])], [np.array([[0.5, 1, 2, 3]])],
                [np.array([[0, np.nan, 2, 3]])], [np.array([[-1, 1, 2, 3]])]):
        with pytest.raises(ValueError):
            est.fit(bad)
    with pytest.raises(ValueError):
        vg.GaussianVoxelizer(grid_size=(4, 4)).fit(sample_clouds())._shape()
    with pytest.raises(ValueError):
        est.fit(sample_clouds()).inverse_transform(None)
    with pytest.raises(ValueError):
        vg.GaussianVoxelizer(box="per-sample").fit(sample_clouds()).inverse_transform(
            np.zeros((1, 1, 4, 4, 4), np.float32))


def test_synth_configs_follow_baseline():
    c0, c3, c4 = synth.CONFIGS[0], synth.CONFIGS[3], synth.CONFIGS[4]
    assert c0.shape == (32, 32, 32) and c0.channels == 5 and c0.n_molecules == 64
    assert abs(sum(c3.element_p) - 1.0) < 1e-12 and c3.channels == 8
    for cfg, lo, hi in ((c0, 9, 29), (c4, 5, 200)):
        pb = synth.packed_batch(cfg, range(200))
        counts = np.diff(pb.offsets)
        assert counts.min() >= lo and counts.max() <= hi
        for b in range(20):
            _, xyz = pb.molecule(b)
            d = np.sqrt(((xyz[:, None] - xyz[None]) ** 2).sum(-1))
            assert d[np.triu_indices(len(xyz), 1)].min() >= cfg.min_dist
    pb = synth.packed_batch(c3, [0])
    assert 1500 <= pb.n_molecules * 0 + len(pb.channels) <= 3000


def test_vectorised_batch_host_path_matches_per_molecule_semantics():
    """generate_batch's vectorised validation, packing and per-molecule boxes
    give the per-molecule results (reference gridgen.py:114-127, 173-221,
    core.py:283-312) on a mixed batch: bad channels, empty sets, a single
    atom, huge coordinates."""
    rng = np.random.default_rng(11)
    spec = vg.GridSpec((10, 12, 14), 3, vg.BoundingBox((0, 0, 0), (5, 5, 5)), 0.4)
    sets = []
    for b in range(200):
        n = int(rng.integers(0, 9))
        ch = rng.integers(0, 3, n)
        if b % 37 == 5 and n:
            ch[0] = 7            # out-of-range channel
        sets.append(vg.ParticleSet(ch, rng.normal(2.5, 3.0, (n, 3))))
    sets.append(vg.ParticleSet([0], [[1e300, -1e300, 0.0]]))
    errors = gridgen._batch_errors(sets, spec)
    slow = {b: e for b, ps in enumerate(sets)
            if (e := gridgen._consistency_error(ps, spec)) is not None}
    assert sorted(errors) == sorted(slow)
    assert all(str(errors[b]) == str(slow[b]) for b in slow)
    offsets, ch, xyz, counts = gridgen.pack_particle_sets(sets, spec, errors)
    for b, ps in enumerate(sets):
        lo, hi = offsets[b], offsets[b + 1]
        if b in errors:
            assert hi == lo
        else:
            assert np.array_equal(ch[lo:hi], ps.channels) and np.array_equal(xyz[lo:hi], ps.positions)
    errs2 = dict(errors)
    origin, delta, specs = gridgen._bbox_policy(sets, spec, 4.0, errs2)
    assert len(specs) == len(sets)
    for b, ps in enumerate(sets):
        if b in errors:
            continue
        try:
            box = vg.bounding_box_of(ps, 0.4, 4.0)
        except ValueError:
            assert b in errs2
            continue
        assert b not in errs2
        assert specs[b].box == box
        assert tuple(origin[b]) == box.origin
        assert tuple(delta[b]) == (box.extents[0] / 12, box.extents[1] / 10, box.extents[2] / 14)


def test_atom_counts_match_generated_molecules_and_cost_shards():
    from paper_2211_08506_b200 import shard, synth

    for k in (0, 4):
        cfg = synth.CONFIGS[k]
        idx = range(10, 30)
        pb = synth.packed_batch(cfg, idx)
        assert np.array_equal(synth.atom_counts(cfg, idx), np.diff(pb.offsets))
    cfg = synth.CONFIGS[4]
    costs = shard.molecule_costs(synth.atom_counts(cfg, range(512)), cfg.grid_bytes,
                                 shard.BYTES_PER_ATOM)
    plan = shard.plan_shards(costs, 8)
    assert plan[0][0] == 0 and plan[-1][1] == 512
    assert all(a[1] == b[0] for a, b in zip(plan, plan[1:]))
    per = [costs[a:b].sum() for a, b in plan]
    assert max(per) / min(per) < 1.05
