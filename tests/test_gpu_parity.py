"""Parity of the sm_100a path against the reference (golden fixtures made by
the real reference) and against the CPU oracle on the same seeded inputs.

The bar is bit-exact float32 grids (which implies the north_star tolerance
|gpu - ref| <= 1e-6 + 1e-5 |ref|, reported on failure) and identical
GenStats counters. Every call goes through the C-ABI library.
"""

from __future__ import annotations

import numpy as np
import pytest

from _golden import (assert_bitwise, config_records, erf_cases, grid_cases, packed_sha, sha,
                     table_cases)
from oracle import voxgrid_oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import synth  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    vg._native.lib()
    yield
    torch.cuda.synchronize()


def spec_of(cfg):
    return vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                       cfg.sigma)


def geom_of(cfg):
    return orc.Geometry(cfg.shape, cfg.channels, cfg.box_origin, cfg.box_extents, cfg.sigma)


# ---------------------------------------------------------------------------
# numerics
# ---------------------------------------------------------------------------
def test_device_erf_matches_golden():
    t, e = erf_cases()
    got = vg.erf_approx(t)
    assert np.array_equal(got.view(np.uint32), e.view(np.uint32))


def test_device_erf_all_floats_0_to_6_vs_oracle():
    hi = int(np.float32(6.0).view(np.uint32))
    step = 1 << 25
    for s in range(0, hi + 1, step):
        bits = torch.arange(s, min(s + step, hi + 1), dtype=torch.int64, device="cuda")
        t = bits.to(torch.int32).view(torch.float32)
        got = vg.erf_approx(t).cpu().numpy()
        tn = t.cpu().numpy()
        with np.errstate(all="ignore"):
            ref = orc.erf_f32(tn)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), hex(s)
        neg = vg.erf_approx(-t).cpu().numpy()
        assert np.array_equal(neg, -got)


@pytest.mark.parametrize("case", range(len(table_cases())))
def test_axis_tables_match_golden(case):
    meta, values = table_cases()[case]
    tabs = vg.fused_axis_tables(meta["mus"], meta["params"], meta["sigma"],
                                threshold=meta["threshold"], periodic=meta["periodic"])
    for a in range(3):
        assert np.array_equal(tabs[a].values.view(np.uint32), values[a].view(np.uint32)), (case, a)
        assert list(tabs[a].support) == meta["supports"][a], (case, a)


# K1 open-axis window search (exact saturation boundaries, multi-pass windows
# wider than the 32-edge buffer, empty windows, one-edge jumps, thresholds,
# per-molecule origins/deltas) against the oracle's full-row restatement.
@pytest.mark.parametrize("sigma,shape,extent,thr", [
    (0.5, (33, 64, 40), 12.0, None),     # typical window, odd counts
    (3.0, (300, 257, 520), 15.0, None),  # windows of hundreds of edges
    (0.004, (20, 17, 9), 10.0, None),    # window shorter than one edge
    (0.7, (31, 65, 129), 20.0, 1e-4),    # threshold
    (0.7, (31, 65, 129), 20.0, -1.0),    # negative threshold keeps zeros
])
@pytest.mark.parametrize("lanes", [None, "2", "4", "8"])
def test_axis_tables_window_search_vs_oracle(sigma, shape, extent, thr, lanes, monkeypatch):
    if lanes is not None:
        monkeypatch.setenv("VG_K1T", lanes)   # K1 lanes per row (default: by batch size)
    rng = np.random.default_rng(int(sigma * 1000) + shape[0])
    n_mol, per = 7, 111
    n = n_mol * per
    offsets = np.arange(0, n + 1, per, dtype=np.int64)
    xyz = rng.uniform(-0.5 * extent, 1.5 * extent, size=(n, 3))   # many far outside
    xyz[::17] = np.round(xyz[::17] * 4) / 4                        # edge-aligned centres
    H, W, D = shape
    spec = vg.GridSpec(shape, 1, vg.BoundingBox((0.0, 0.0, 0.0), (extent,) * 3), sigma)
    mo = rng.uniform(-2.0, 2.0, size=(n_mol, 3))
    md = np.array([[extent / W, extent / H, extent / D]]) * rng.uniform(0.8, 1.25, size=(n_mol, 1))
    for per_mol in (False, True):
        kw = {"mol_origin": mo, "mol_delta": md} if per_mol else {}
        tx, ty, tz, sup = vg.axis_tables_batch(offsets, np.zeros(n, np.int32), xyz, spec,
                                               threshold=thr, **kw)
        got = [t.cpu().numpy() for t in (tx, ty, tz)]
        sup = sup.cpu().numpy()
        for a, cnt in enumerate((W, H, D)):
            for b in range(n_mol):
                o = mo[b, a] if per_mol else 0.0
                d = md[b, a] if per_mol else extent / cnt
                rows = slice(offsets[b], offsets[b + 1])
                ref, rsup = orc.axis_tables(xyz[rows, a], cnt, o, d, sigma, threshold=thr)
                assert np.array_equal(got[a][rows].view(np.uint32), ref.view(np.uint32)), \
                    (per_mol, a, b)
                assert np.array_equal(sup[rows, a], rsup), (per_mol, a, b)


# ---------------------------------------------------------------------------
# single grids: the reference's KAT-style cases
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("idx", range(len(grid_cases())))
def test_generate_grid_matches_golden(idx):
    m, g = grid_cases()[idx]
    lattice = vg.LatticeCell(tuple(m["periodic"])) if m["periodic"] else None
    spec = vg.GridSpec(tuple(m["shape"]), m["channels"],
                       vg.BoundingBox(tuple(m["origin"]), tuple(m["extents"])), m["sigma"],
                       lattice)
    ps = vg.ParticleSet(np.array(m["chans"], dtype=np.int64),
                        np.array(m["pos"]).reshape(-1, 3), lattice)
    grid, st = vg.generate_grid(ps, spec, mode=m["mode"], threshold=m["threshold"])
    assert grid.data.is_cuda and grid.data.dtype == torch.float32
    assert_bitwise(grid.numpy(), g, m["name"])
    assert (st.voxel_writes, st.erf_evals, st.nonzero_voxels) == (
        m["voxel_writes"], m["erf_evals"], m["nonzero_voxels"]), m["name"]


def test_layout_contract_argmax():
    # reference test_core.py:131-142
    spec = vg.GridSpec((2, 3, 4), 1, vg.BoundingBox((0, 0, 0), (3, 2, 4)), 0.08)
    grid, _ = vg.generate_grid(vg.ParticleSet([0], [[2.5, 0.5, 3.5]]), spec)
    data = grid.numpy()
    assert data.shape == (1, 2, 3, 4)
    assert np.unravel_index(np.argmax(data), data.shape) == (0, 0, 2, 3)
    assert grid.value_at(0, (2, 0, 3)) == data[0, 0, 2, 3]


# ---------------------------------------------------------------------------
# BASELINE configs: golden hashes from the real reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("rec_i", range(len(config_records()["batches"])))
def test_config_batches_match_golden(rec_i):
    rec = config_records()["batches"][rec_i]
    cfg = synth.CONFIGS[rec["config"]]
    pb = synth.packed_batch(cfg, rec["indices"])
    assert packed_sha(pb) == rec["inputs_sha"]
    spec = spec_of(cfg)
    if rec["spec_policy"] == "fixed":
        grids, stats = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
        stats = stats.cpu().numpy()
        host = grids.cpu().numpy()
        for b, g in enumerate(rec["grids"]):
            assert sha(host[b]) == g["sha"], (rec["config"], rec["indices"][b])
            assert stats[b, 0] == g["voxel_writes"] and stats[b, 1] == g["nonzero_voxels"]
    else:
        sets = [vg.ParticleSet(*pb.molecule(b)) for b in range(pb.n_molecules)]
        res = vg.generate_batch(sets, spec, spec_policy=rec["spec_policy"])
        assert not res.errors
        for (grid, st), g in zip(res.results, rec["grids"]):
            assert [list(grid.spec.box.origin), list(grid.spec.box.extents)] == g["box"]
            assert sha(grid.numpy()) == g["sha"]
            assert (st.voxel_writes, st.erf_evals, st.nonzero_voxels) == (
                g["voxel_writes"], g["erf_evals"], g["nonzero_voxels"])


def test_estimator_matches_golden():
    from paper_2211_08506_b200 import GaussianVoxelizer

    rec = config_records()["estimator"]
    clouds = []
    for b in range(6):
        ch, xyz = synth.molecule(synth.CONFIGS[0], b)
        clouds.append(np.column_stack([ch.astype(np.float64), xyz]))
    est = GaussianVoxelizer(grid_size=24, sigma=0.4).fit(clouds)
    assert est.channels_ == rec["shared"]["channels"]
    assert [list(est.box_.origin), list(est.box_.extents)] == rec["shared"]["box"]
    out = est.transform(clouds)
    assert out.is_cuda and tuple(out.shape) == (6, est.channels_, 24, 24, 24)
    host = out.cpu().numpy()
    assert [sha(g) for g in host] == rec["shared"]["shas"]
    per = GaussianVoxelizer(grid_size=(20, 16, 12), sigma=0.5, box="per-sample").fit(clouds)
    assert [sha(g) for g in per.transform(clouds).cpu().numpy()] == rec["per_sample"]["shas"]


# ---------------------------------------------------------------------------
# full configs vs the oracle on this host
# ---------------------------------------------------------------------------
def _compare_with_oracle(cfg, indices, workers=None):
    pb = synth.packed_batch(cfg, indices)
    grids, stats = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec_of(cfg))
    ref, ref_stats = orc.batch(pb.offsets, pb.channels, pb.xyz, geom_of(cfg),
                               workers=workers or orc.host_cores())
    assert_bitwise(grids.cpu().numpy(), ref, cfg.name)
    st = stats.cpu().numpy()
    assert [int(v) for v in st[:, 0]] == [r["voxel_writes"] for r in ref_stats]
    assert [int(v) for v in st[:, 1]] == [r["nonzero_voxels"] for r in ref_stats]


def test_cfg0_full_vs_oracle():
    _compare_with_oracle(synth.CONFIGS[0], range(64))


def test_cfg1_full_vs_oracle():
    cfg = synth.CONFIGS[1]
    for start in range(0, cfg.n_molecules, 256):
        _compare_with_oracle(cfg, range(start, start + 256))


def test_cfg2_full_vs_oracle():
    # all 65,536 grids (2.1 G voxels), in chunks of 4096 molecules
    cfg = synth.CONFIGS[2]
    for start in range(0, cfg.n_molecules, 4096):
        _compare_with_oracle(cfg, range(start, start + 4096))


def test_cfg3_full_vs_oracle():
    cfg = synth.CONFIGS[3]
    for start in range(0, cfg.n_molecules, 8):
        _compare_with_oracle(cfg, range(start, start + 8))


def test_cfg4_full_vs_oracle():
    cfg = synth.CONFIGS[4]
    for start in range(0, cfg.n_molecules, 1024):
        _compare_with_oracle(cfg, range(start, start + 1024))


# ---------------------------------------------------------------------------
# size-independent properties at full size
# ---------------------------------------------------------------------------
def _digest(t):
    flat = t.reshape(t.shape[0], -1).view(torch.int32).to(torch.int64)
    w = torch.arange(1, flat.shape[1] + 1, device=t.device, dtype=torch.int64)
    return ((flat * w).sum(dim=1) % (2**61 - 1)).cpu().numpy()


def test_cfg2_full_chunking_invariant_and_nonzero_counts():
    """All 65,536 cfg2 grids: per-grid digests are identical whether the batch
    is launched in chunks of 8192 or 5000 molecules (output independent of
    launch shape), and the kernel's nonzero counters equal torch's count."""
    cfg = synth.CONFIGS[2]
    pb = synth.packed_batch(cfg)
    spec = spec_of(cfg)

    def run(chunk):
        digs, nz = [], []
        for s in range(0, pb.n_molecules, chunk):
            e = min(s + chunk, pb.n_molecules)
            lo, hi = pb.offsets[s], pb.offsets[e]
            g, st = vg.generate_packed(pb.offsets[s:e + 1] - lo, pb.channels[lo:hi],
                                       pb.xyz[lo:hi], spec)
            digs.append(_digest(g))
            cnt = (g.reshape(e - s, -1) != 0).sum(dim=1).cpu().numpy()
            assert np.array_equal(cnt, st[:, 1].cpu().numpy())
            nz.append(cnt)
            del g
        return np.concatenate(digs), np.concatenate(nz)

    d1, n1 = run(8192)
    d2, n2 = run(5000)
    assert np.array_equal(d1, d2) and np.array_equal(n1, n2)


def test_normalization_with_margin():
    # reference acceptance c01 (test_acceptance.py:59-74): mass == atom count
    rng = np.random.default_rng(20240817)
    for trial in range(20):
        sigma = float(rng.choice([0.05, 0.1, 0.25, 0.5]))
        ext = float(rng.uniform(7.0, 12.0))
        origin = rng.uniform(-3, 3, 3)
        n = int(rng.integers(1, 9))
        pos = origin + 2.0 + rng.uniform(0, ext - 4.0, (n, 3))
        ch = rng.integers(0, 3, n)
        spec = vg.GridSpec((24, 24, 24), 3, vg.BoundingBox(tuple(origin), (ext,) * 3), sigma)
        grid, _ = vg.generate_grid(vg.ParticleSet(ch, pos), spec)
        sums = grid.channel_sums()
        counts = np.bincount(ch, minlength=3)
        assert abs(sums.sum() - n) <= 1e-3 * n
        for c in range(3):
            assert abs(sums[c] - counts[c]) <= max(1e-3 * counts[c], 1e-6)


def test_translation_equivariance_bitwise():
    spec = vg.GridSpec((16, 16, 16), 1, vg.BoundingBox((0, 0, 0), (8, 8, 8)), 0.5)
    base_pos = np.array([[2.25, 3.5, 4.125], [5.0, 2.75, 6.5]])
    base, _ = vg.generate_grid(vg.ParticleSet([0, 0], base_pos), spec)
    for shift in [(1.5, -2.25, 4.0), (0.1, 0.37, -1.234), (-2.9, 1.7, 0.3)]:
        moved = vg.GridSpec((16, 16, 16), 1, spec.box.translate(shift), 0.5)
        g, _ = vg.generate_grid(vg.ParticleSet([0, 0], base_pos + np.asarray(shift)), moved)
        assert torch.equal(g.data, base.data)


# ---------------------------------------------------------------------------
# edge cases and errors
# ---------------------------------------------------------------------------
def test_empty_batch_and_empty_molecules():
    spec = vg.GridSpec((8, 8, 8), 2, vg.BoundingBox((0, 0, 0), (4, 4, 4)), 0.3)
    res = vg.generate_batch([], spec)
    assert tuple(res.tensor.shape) == (0, 2, 8, 8, 8)
    sets = [vg.ParticleSet.from_rows([]), vg.ParticleSet([1], [[2, 2, 2]]),
            vg.ParticleSet.from_rows([])]
    res = vg.generate_batch(sets, spec)
    assert not res.errors
    t = res.tensor.cpu().numpy()
    assert not t[0].any() and not t[2].any() and t[1, 1].sum() > 0.99
    ref, _ = orc.grid([1], [[2, 2, 2]], orc.Geometry((8, 8, 8), 2, (0, 0, 0), (4, 4, 4), 0.3))
    assert_bitwise(t[1], ref)


def test_per_index_errors_do_not_abort_batch():
    spec = vg.GridSpec((8, 8, 8), 1, vg.BoundingBox((0, 0, 0), (4, 4, 4)), 0.3)
    good = vg.ParticleSet([0], [[2, 2, 2]])
    bad = vg.ParticleSet([5], [[2, 2, 2]])
    res = vg.generate_batch([good, bad, good], spec)
    assert list(res.errors) == [1]
    assert res.results[0] is not None and res.results[2] is not None and res.results[1] is None
    assert not res.tensor[1].any()
    with pytest.raises(ValueError):
        res.grids()
    with pytest.raises(ValueError):
        vg.generate_grid(bad, spec)


def test_periodicity_mismatch_errors():
    cell = vg.LatticeCell((6.0, 6.0, 6.0))
    spec = vg.GridSpec((8, 8, 8), 1, vg.BoundingBox((0, 0, 0), (6, 6, 6)), 0.3, cell)
    with pytest.raises(ValueError):
        vg.generate_grid(vg.ParticleSet([0], [[1, 1, 1]]), spec)
    open_spec = vg.GridSpec((8, 8, 8), 1, vg.BoundingBox((0, 0, 0), (6, 6, 6)), 0.3)
    with pytest.raises(ValueError):
        vg.generate_grid(vg.ParticleSet([0], [[1, 1, 1]], cell), open_spec)


def test_dense_mode_counts_and_bits():
    spec = vg.GridSpec((16, 16, 16), 1, vg.BoundingBox((0, 0, 0), (6, 6, 6)), 0.2)
    rng = np.random.default_rng(19)
    ps = vg.ParticleSet(np.zeros(5, int), rng.uniform(0, 6, (5, 3)))
    gs, ss = vg.generate_grid(ps, spec, mode="sparse")
    gd, sd = vg.generate_grid(ps, spec, mode="dense")
    assert torch.equal(gs.data, gd.data)
    assert sd.voxel_writes == 5 * 16**3 and ss.voxel_writes <= sd.voxel_writes
    with pytest.raises(ValueError):
        vg.generate_grid(ps, spec, mode="fast")
    with pytest.raises(ValueError):
        vg.generate_grid(ps, spec, dtype=np.float64)


def test_candidate_list_overflow_path_vs_oracle():
    """A 3000-atom single-channel molecule in a small box: every y-chunk has
    > 1024 candidate atoms, exercising the segmented list path."""
    rng = np.random.default_rng(5)
    n = 3000
    xyz = rng.uniform(0, 6, (n, 3))
    ch = np.zeros(n, np.int32)
    ch[::7] = 1
    spec = vg.GridSpec((20, 24, 28), 2, vg.BoundingBox((0, 0, 0), (6, 6, 6)), 0.6)
    grids, st = vg.generate_packed(np.array([0, n]), ch, xyz, spec)
    ref, rs = orc.grid(ch, xyz, orc.Geometry((20, 24, 28), 2, (0, 0, 0), (6, 6, 6), 0.6))
    assert_bitwise(grids[0].cpu().numpy(), ref, "overflow")
    assert int(st[0, 0]) == rs["voxel_writes"] and int(st[0, 1]) == rs["nonzero_voxels"]


@pytest.mark.parametrize("policy", ["fixed", "per-molecule-bbox"])
def test_candidate_bins_vs_oracle_and_unbinned(policy, monkeypatch):
    """K2 bins (large molecules): mixed sizes incl. empty and tiny molecules,
    atoms outside the box, 3 channels, odd shape; equal to the oracle and to
    the unbinned scan path (VG_BINS=0)."""
    rng = np.random.default_rng(17)
    sizes = [1400, 0, 3, 900, 2100, 700]
    sets = []
    for n in sizes:
        xyz = rng.normal(6.0, 2.5, size=(n, 3))
        sets.append(vg.ParticleSet(rng.integers(0, 3, size=n), xyz))
    spec = vg.GridSpec((37, 30, 44), 3, vg.BoundingBox((0, 0, 0), (12, 12, 12)), 0.45)
    got = vg.generate_batch(sets, spec, spec_policy=policy)
    monkeypatch.setenv("VG_BINS", "0")
    plain = vg.generate_batch(sets, spec, spec_policy=policy)
    monkeypatch.delenv("VG_BINS")
    a, b = got.tensor.cpu().numpy(), plain.tensor.cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert plain.errors.keys() == got.errors.keys()
    for i, ps in enumerate(sets):
        if i in got.errors:
            continue
        g, st = got.results[i]
        sp = g.spec
        ref, rs = orc.grid(np.asarray(ps.channels), np.asarray(ps.positions),
                           orc.Geometry(sp.shape, 3, sp.box.origin, sp.box.extents, 0.45))
        assert_bitwise(a[i], ref, f"bins {policy} {i}")
        assert st.voxel_writes == rs["voxel_writes"] and st.nonzero_voxels == rs["nonzero_voxels"]


@pytest.mark.parametrize("env", [{}, {"VG_FUSE": "0"}, {"VG_GXWIN": "0"}, {"VG_FUSE": "1", "VG_SW": "4"}])
def test_many_channels_threshold_paths_vs_oracle(env, monkeypatch):
    """Small molecules over 12 channels with a threshold: the channel-fused
    path (default), per-channel CTAs, full-tile gx staging and float4 slots
    all match the oracle bit for bit."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(123)
    sizes = rng.integers(1, 40, size=23)
    sizes[5] = 0
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offsets[-1])
    xyz = rng.uniform(-1.0, 9.0, (n, 3))
    ch = rng.integers(0, 12, n).astype(np.int32)
    shape = (36, 28, 40)
    spec = vg.GridSpec(shape, 12, vg.BoundingBox((0, 0, 0), (8.0, 8.0, 8.0)), 0.4)
    grids, st = vg.generate_packed(offsets, ch, xyz, spec, threshold=1e-3)
    ref, rs = orc.batch(offsets, ch, xyz, orc.Geometry(shape, 12, (0, 0, 0), (8.0, 8.0, 8.0), 0.4),
                        threshold=1e-3, workers=orc.host_cores())
    assert_bitwise(grids.cpu().numpy(), ref, f"many channels {env}")
    assert [int(v) for v in st[:, 0].cpu()] == [r["voxel_writes"] for r in rs]
    assert [int(v) for v in st[:, 1].cpu()] == [r["nonzero_voxels"] for r in rs]


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 7), (5, 3, 4), (33, 31, 36), (4, 70, 8)])
def test_odd_shapes_vs_oracle(shape):
    rng = np.random.default_rng(sum(shape))
    n = 9
    ext = (3.0, 2.5, 4.0)
    xyz = rng.uniform(-0.5, 4.0, (n, 3))
    ch = rng.integers(0, 3, n).astype(np.int32)
    spec = vg.GridSpec(shape, 3, vg.BoundingBox((0, 0, 0), ext), 0.35)
    grids, st = vg.generate_packed(np.array([0, 4, n]), ch, xyz, spec)
    geom = orc.Geometry(shape, 3, (0, 0, 0), ext, 0.35)
    ref, rs = orc.batch(np.array([0, 4, n]), ch, xyz, geom)
    assert_bitwise(grids.cpu().numpy(), ref, str(shape))
    assert [int(v) for v in st[:, 1].cpu()] == [r["nonzero_voxels"] for r in rs]


def test_out_tensor_and_stream():
    cfg = synth.CONFIGS[0]
    pb = synth.packed_batch(cfg, range(4))
    spec = spec_of(cfg)
    out = torch.full((4, 5, 32, 32, 32), 7.0, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec, out=out, with_stats=False)
    s.synchronize()
    ref, _ = orc.batch(pb.offsets, pb.channels, pb.xyz, geom_of(cfg))
    assert_bitwise(out.cpu().numpy(), ref, "out=")


def test_generic_kernel_matches_golden(monkeypatch):
    """The fallback slab kernel (any shape, VG_FORCE_GENERIC=1) stays bit-exact."""
    monkeypatch.setenv("VG_FORCE_GENERIC", "1")
    for m, g in grid_cases():
        lattice = vg.LatticeCell(tuple(m["periodic"])) if m["periodic"] else None
        spec = vg.GridSpec(tuple(m["shape"]), m["channels"],
                           vg.BoundingBox(tuple(m["origin"]), tuple(m["extents"])), m["sigma"],
                           lattice)
        ps = vg.ParticleSet(np.array(m["chans"], dtype=np.int64),
                            np.array(m["pos"]).reshape(-1, 3), lattice)
        grid, st = vg.generate_grid(ps, spec, mode=m["mode"], threshold=m["threshold"])
        assert_bitwise(grid.numpy(), g, m["name"])
        assert st.nonzero_voxels == m["nonzero_voxels"]
    _compare_with_oracle(synth.CONFIGS[1], range(64))


@pytest.mark.parametrize("sw", ["1", "4"])
def test_slot_width_variants_match_golden(monkeypatch, sw):
    """The row kernel's narrower slot layouts (VG_SW) stay bit-exact."""
    monkeypatch.setenv("VG_SW", sw)
    for m, g in grid_cases():
        lattice = vg.LatticeCell(tuple(m["periodic"])) if m["periodic"] else None
        spec = vg.GridSpec(tuple(m["shape"]), m["channels"],
                           vg.BoundingBox(tuple(m["origin"]), tuple(m["extents"])), m["sigma"],
                           lattice)
        ps = vg.ParticleSet(np.array(m["chans"], dtype=np.int64),
                            np.array(m["pos"]).reshape(-1, 3), lattice)
        grid, st = vg.generate_grid(ps, spec, mode=m["mode"], threshold=m["threshold"])
        assert_bitwise(grid.numpy(), g, m["name"])
        assert st.nonzero_voxels == m["nonzero_voxels"]
    _compare_with_oracle(synth.CONFIGS[4], range(0, 4096, 41))
    _compare_with_oracle(synth.CONFIGS[3], [3])


def test_pipeline_matches_serial_path():
    """GridPipeline (copy / tables / compute streams, double buffers) gives
    the serial path's bits for host and device inputs, across slot reuse."""
    from paper_2211_08506_b200.loader import GridPipeline, pinned_csr

    cfg = synth.CONFIGS[4]
    spec = spec_of(cfg)
    batches = [synth.packed_batch(cfg, range(s, s + n)) for s, n in ((0, 7), (40, 13), (99, 5))]
    refs = []
    for pb in batches:
        g, st = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
        refs.append((g.cpu().numpy(), st.cpu().numpy()))
    pipe = GridPipeline(spec)
    outs = []
    for rnd in range(2):
        for pb, (g_ref, st_ref) in zip(batches, refs):
            if rnd == 0:
                res = pipe.submit(*pinned_csr(pb.offsets, pb.channels, pb.xyz))
            else:
                res = pipe.submit(torch.from_numpy(pb.offsets).cuda(),
                                  torch.from_numpy(pb.channels).cuda(),
                                  torch.from_numpy(pb.xyz).cuda())
            res.ready.synchronize()
            outs.append((res.grids.cpu().numpy(), res.stats.cpu().numpy(), g_ref, st_ref))
    for g, st, g_ref, st_ref in outs:
        assert_bitwise(g, g_ref, "pipeline")
        assert np.array_equal(st, st_ref)


def test_pipeline_back_to_back_with_stats_readback():
    """Submissions queued without host syncs (depth-3 slots), host inputs as
    pinned tensors and plain numpy, stats read back into pinned host memory
    by the same native call: bits equal the serial path."""
    from paper_2211_08506_b200.loader import GridPipeline, pinned_csr

    cfg = synth.CONFIGS[4]
    spec = spec_of(cfg)
    batches = [synth.packed_batch(cfg, range(s, s + n)) for s, n in ((3, 9), (70, 4), (200, 11))]
    pipe = GridPipeline(spec, depth=3)
    res, st_host = [], []
    for i, pb in enumerate(batches):
        st_h = torch.empty((pb.n_molecules, 2), dtype=torch.int64).pin_memory()
        inputs = pinned_csr(pb.offsets, pb.channels, pb.xyz) if i % 2 == 0 else (
            pb.offsets, pb.channels, pb.xyz)
        res.append(pipe.submit(*inputs, stats_out=st_h))
        st_host.append(st_h)
    pipe.synchronize()
    for pb, r, st_h in zip(batches, res, st_host):
        g_ref, s_ref = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
        assert_bitwise(r.grids.cpu().numpy(), g_ref.cpu().numpy(), "pipeline b2b")
        assert np.array_equal(st_h.numpy(), s_ref.cpu().numpy())


@pytest.mark.parametrize("yp", ["1", "2"])
def test_slab_pair_hot_loop_variants(monkeypatch, yp):
    """Both hot loops (single slabs, slab pairs: VG_YP) are bit-exact: golden
    grids (odd slab counts, periodic, thresholds), the segmented overflow
    path (continued sums), K2 bins, fused and per-channel CTAs."""
    monkeypatch.setenv("VG_YP", yp)
    for m, g in grid_cases():
        lattice = vg.LatticeCell(tuple(m["periodic"])) if m["periodic"] else None
        spec = vg.GridSpec(tuple(m["shape"]), m["channels"],
                           vg.BoundingBox(tuple(m["origin"]), tuple(m["extents"])), m["sigma"],
                           lattice)
        ps = vg.ParticleSet(np.array(m["chans"], dtype=np.int64),
                            np.array(m["pos"]).reshape(-1, 3), lattice)
        grid, st = vg.generate_grid(ps, spec, mode=m["mode"], threshold=m["threshold"])
        assert_bitwise(grid.numpy(), g, m["name"])
        assert st.nonzero_voxels == m["nonzero_voxels"]
    test_candidate_list_overflow_path_vs_oracle()
    _compare_with_oracle(synth.CONFIGS[1], range(0, 1024, 9))
    _compare_with_oracle(synth.CONFIGS[4], range(0, 4096, 37))
    _compare_with_oracle(synth.CONFIGS[3], [5, 17])
    monkeypatch.setenv("VG_FUSE", "0")
    _compare_with_oracle(synth.CONFIGS[0], range(64))


@pytest.mark.parametrize("env", [{"VG_TAPER": "2", "VG_TASK_KB": "1024"},
                                 {"VG_TAPER": "2", "VG_TASK_KB": "1024", "VG_BULK": "0"},
                                 {"VG_TAPER": "0"}, {"VG_BULK": "0"}])
def test_tapered_tail_and_staging_variants_vs_oracle(env, monkeypatch):
    """The launch's tapered tail (the last molecules in quarter-length
    y-chunks; VG_TAPER=2 forces it on small batches, a third of the molecules,
    VG_TASK_KB keeps the full-size tiles the taper divides)
    and both staging paths (bulk copies / cp.async: VG_BULK) are bit-exact vs
    the oracle on fused batches, incl. large molecules that fall back to
    per-channel passes, with identical counters."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _compare_with_oracle(synth.CONFIGS[1], range(0, 1024, 17))
    _compare_with_oracle(synth.CONFIGS[0], range(64))
    _compare_with_oracle(synth.CONFIGS[4], range(0, 4096, 29))


def test_fused_cta_fallback_on_large_molecules_vs_oracle(monkeypatch):
    """Channel-fused CTAs on molecules too large for one staging pass fall
    back to the per-channel path (halved sub-chunks, segmented slabs);
    VG_FUSE=1 forces fused CTAs on these sizes."""
    monkeypatch.setenv("VG_FUSE", "1")
    rng = np.random.default_rng(2024)
    sizes = [3, 150, 400, 0, 60, 900, 210]
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offsets[-1])
    xyz = rng.uniform(0.0, 10.0, (n, 3))
    ch = rng.choice(4, size=n, p=[0.5, 0.3, 0.15, 0.05]).astype(np.int32)
    shape = (40, 36, 48)
    spec = vg.GridSpec(shape, 4, vg.BoundingBox((0, 0, 0), (10.0, 10.0, 10.0)), 0.5)
    grids, st = vg.generate_packed(offsets, ch, xyz, spec)
    ref, rs = orc.batch(offsets, ch, xyz, orc.Geometry(shape, 4, (0, 0, 0), (10.0, 10.0, 10.0), 0.5),
                        workers=orc.host_cores())
    assert_bitwise(grids.cpu().numpy(), ref, "fused halving")
    assert [int(v) for v in st[:, 0].cpu()] == [r["voxel_writes"] for r in rs]
    assert [int(v) for v in st[:, 1].cpu()] == [r["nonzero_voxels"] for r in rs]


def test_estimator_packed_fast_path_equals_per_sample_path():
    """transform's batch-at-once validation and packing (fixed box) gives the
    per-sample path's bits, empty samples included; a sample with an
    out-of-range channel still raises the reference's ValueError."""
    rng = np.random.default_rng(77)
    X = []
    for i in range(40):
        n = int(rng.integers(0, 12))
        X.append(np.column_stack([rng.integers(0, 3, n), rng.uniform(0, 6, (n, 3))]))
    X[7] = np.zeros((0, 4))
    est = vg.GaussianVoxelizer(grid_size=(20, 18, 24), sigma=0.45, n_channels=3,
                               box=((0.0, 0.0, 0.0), (6.0, 6.0, 6.0))).fit(X)
    fast = est.transform(X)
    slow = vg.generate_batch(est._sets(X), est._spec()).tensor
    assert np.array_equal(fast.cpu().numpy().view(np.uint32), slow.cpu().numpy().view(np.uint32))
    bad = list(X)
    bad[3] = np.array([[5.0, 1.0, 1.0, 1.0]])
    with pytest.raises(ValueError):
        est.transform(bad)


def test_transform_back_to_back_calls_recycle_outputs_safely():
    """Consecutive transform calls whose outputs are consumed on the caller's
    stream or a side stream (a device-side digest, then dropped, no host sync):
    the caching allocator recycles the outputs across calls while the pipeline's
    compute streams write them, and every digest still equals the serial path's."""
    cfg = synth.CONFIGS[0]
    spec = spec_of(cfg)
    est = None
    want, got = [], []
    side = torch.cuda.Stream()
    for k in range(14):
        n = (48, 48, 17, 48, 64, 48)[k % 6]
        pb = synth.packed_batch(cfg, range(70 * k, 70 * k + n))
        X = [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
             for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
        if est is None:
            est = vg.GaussianVoxelizer(grid_size=cfg.shape, sigma=cfg.sigma,
                                       n_channels=cfg.channels,
                                       box=(cfg.box_origin, cfg.box_extents)).fit(X)
        g = est.transform(X)
        if k % 3 == 2:   # a consumer on another stream, ordered after the caller's
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                got.append(g.view(torch.int32).sum(dim=(1, 2, 3, 4), dtype=torch.int64))
            g.record_stream(side)
        else:
            got.append(g.view(torch.int32).sum(dim=(1, 2, 3, 4), dtype=torch.int64))
        del g
        ref, _ = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
        want.append(ref.view(torch.int32).sum(dim=(1, 2, 3, 4), dtype=torch.int64))
        del ref
    torch.cuda.synchronize()
    for k, (a, b) in enumerate(zip(got, want)):
        assert torch.equal(a.cpu(), b.cpu()), k


def test_transform_chunked_pipeline_equals_single_launch():
    """transform's chunked, pipelined path (loader.generate_rows: pinned
    staging, one GridPipeline submit per chunk into slices of one output)
    gives the single-launch bits for every chunk schedule, empty samples
    included, and the result is usable on the caller's stream without a
    sync; a bad sample in a LATE chunk still raises the reference's error."""
    from paper_2211_08506_b200.loader import generate_rows

    cfg = synth.CONFIGS[0]
    pb = synth.packed_batch(cfg, range(37))
    X = [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
         for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
    X[5] = np.zeros((0, 4))
    X[36] = np.zeros((0, 4))
    spec = spec_of(cfg)
    offs = np.concatenate([[0], np.cumsum([len(x) for x in X])])
    rows = np.concatenate(X)
    ref, _ = vg.generate_packed(offs, rows[:, 0].astype(np.int32), rows[:, 1:4], spec)
    ref = ref.cpu().numpy()
    for first, cap in ((1, 1), (1, 4), (3, 7), (64, 256), (37, 37)):
        got = generate_rows(X, spec, first=first, max_chunk=cap)
        # consumed on the current stream with no explicit synchronisation
        digest = got.view(torch.int32).sum(dim=(1, 2, 3, 4), dtype=torch.int64).cpu().numpy()
        assert np.array_equal(digest, ref.view(np.int32).astype(np.int64).sum(axis=(1, 2, 3, 4)))
        assert_bitwise(got.cpu().numpy(), ref, f"chunks {first}/{cap}")
    est = vg.GaussianVoxelizer(grid_size=cfg.shape, sigma=cfg.sigma, n_channels=cfg.channels,
                               box=(cfg.box_origin, cfg.box_extents)).fit(X)
    assert_bitwise(est.transform(X).cpu().numpy(), ref, "transform")
    assert generate_rows([], spec).shape == (0, 5, 32, 32, 32)
    for late in (30, 36):
        for bad_row in ([[7.0, 1.0, 1.0, 1.0]], [[1.0, np.nan, 1.0, 1.0]], [[0.5, 1, 1, 1]],
                        [[1.0, 1.0, 1.0]]):
            bad = list(X)
            bad[late] = np.array(bad_row)
            assert generate_rows(bad, spec, first=4, max_chunk=8) is None
            with pytest.raises(ValueError):
                est.transform(bad)
    # the pipeline is intact after the failures
    assert_bitwise(est.transform(X).cpu().numpy(), ref, "transform after failures")


@pytest.mark.parametrize("policy", ["fixed", "per-molecule-bbox"])
def test_generate_batch_pipelined_equals_single_launch(policy, monkeypatch):
    """generate_batch over a large batch (> PIPELINE_MIN_BATCH) runs through
    the chunked pipeline (loader.generate_sets); grids, per-molecule GenStats
    and per-index errors equal the single-launch path, with failed and empty
    molecules spread over several chunks."""
    from paper_2211_08506_b200 import gridgen

    cfg = synth.CONFIGS[0]
    spec = spec_of(cfg)
    pb = synth.packed_batch(cfg, range(300))
    sets = [vg.ParticleSet(pb.channels[a:b], pb.xyz.reshape(-1, 3)[a:b])
            for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
    sets[3] = vg.ParticleSet(np.zeros(0, np.int64), np.zeros((0, 3)))
    sets[150] = vg.ParticleSet(np.array([0, 9]), np.ones((2, 3)))      # channel out of range
    sets[299] = vg.ParticleSet(np.array([7]), np.ones((1, 3)))
    import functools

    from paper_2211_08506_b200 import loader

    got = vg.generate_batch(sets, spec, spec_policy=policy)          # one submission
    with monkeypatch.context() as m:                                 # many chunks
        m.setattr(loader, "generate_sets",
                  functools.partial(loader.generate_sets, first=7, max_chunk=50))
        chunked = vg.generate_batch(sets, spec, spec_policy=policy)
    assert_bitwise(chunked.tensor.cpu().numpy(), got.tensor.cpu().numpy(), "chunked sets")
    monkeypatch.setattr(gridgen, "PIPELINE_MIN_BATCH", 1 << 30)
    ref = vg.generate_batch(sets, spec, spec_policy=policy)
    assert sorted(got.errors) == sorted(ref.errors)
    assert {150, 299} <= set(got.errors)
    assert_bitwise(got.tensor.cpu().numpy(), ref.tensor.cpu().numpy(), f"pipelined {policy}")
    for a, b in zip(got.results, ref.results):
        assert (a is None) == (b is None)
        if a is not None:
            assert a[1].voxel_writes == b[1].voxel_writes
            assert a[1].nonzero_voxels == b[1].nonzero_voxels
            assert a[0].spec == b[0].spec


def _small_vs_two_kernel(monkeypatch, offsets, ch, xyz, spec, **kw):
    """The same batch through K13 (VG_SMALL=1) and through K1 + K3
    (VG_SMALL=0): grids bit-identical, counters identical."""
    monkeypatch.setenv("VG_SMALL", "1")
    g1, s1 = vg.generate_packed(offsets, ch, xyz, spec, check=False, **kw)
    g1, s1 = g1.cpu().numpy(), s1.cpu().numpy()
    monkeypatch.setenv("VG_SMALL", "0")
    g0, s0 = vg.generate_packed(offsets, ch, xyz, spec, check=False, **kw)
    assert_bitwise(g1, g0.cpu().numpy(), "K13 vs K1+K3")
    assert np.array_equal(s1, s0.cpu().numpy())
    return g1, s1


@pytest.mark.parametrize("shape", [(32, 32, 32), (20, 18, 24), (7, 9, 12), (64, 64, 64),
                                   (33, 5, 8), (1, 1, 4)])
def test_small_kernel_equals_two_kernel_path(monkeypatch, shape):
    """K13 (one launch: tables in shared memory + gather) against the
    two-kernel path on random batches: shapes, empty molecules, thresholds,
    per-molecule boxes, and molecules with more atoms of one channel than a
    K13 pass holds (several compaction passes)."""
    rng = np.random.default_rng(sum(shape))
    B = 23
    counts = rng.integers(0, 30, B)
    counts[3] = 0
    counts[5] = 300                                    # > one pass (cap <= 64)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    n = int(offsets[-1])
    ch = rng.integers(0, 4, n).astype(np.int32)
    ch[offsets[5]:offsets[6]] = 1                      # all in one channel
    xyz = rng.uniform(-1, 9, (n, 3))
    spec = vg.GridSpec(shape, 4, vg.BoundingBox((0.0, 0.0, 0.0), (8.0, 8.0, 8.0)), 0.45)
    _small_vs_two_kernel(monkeypatch, offsets, ch, xyz, spec)
    _small_vs_two_kernel(monkeypatch, offsets, ch, xyz, spec, threshold=1e-3)
    _small_vs_two_kernel(monkeypatch, offsets, ch, xyz, spec, mode="dense")
    mo = rng.uniform(-2, 1, (B, 3))
    md = rng.uniform(0.1, 0.4, (B, 3))
    _small_vs_two_kernel(monkeypatch, offsets, ch, xyz, spec, mol_origin=mo, mol_delta=md)


def test_small_kernel_flags_invalid_device_atoms(monkeypatch):
    """Device inputs with a channel outside [0, C) or a NaN coordinate: K13
    skips the atom and flags its molecule exactly as K1 + K3 do."""
    cfg = synth.CONFIGS[0]
    pb = synth.packed_batch(cfg, range(6))
    ch = pb.channels.copy()
    xyz = pb.xyz.reshape(-1, 3).copy()
    ch[pb.offsets[1]] = 9
    xyz[pb.offsets[3] + 1, 2] = np.nan
    off_d, ch_d, xyz_d = (torch.from_numpy(a).cuda() for a in (pb.offsets, ch, xyz))
    g, st = _small_vs_two_kernel(monkeypatch, off_d, ch_d, xyz_d, spec_of(cfg))
    assert list(np.flatnonzero(st[:, 0] < 0)) == [1, 3]


def test_small_batches_take_the_one_launch_path(monkeypatch):
    """A handful of cfg0 molecules (a few MB of grids) launch one kernel
    (K13) instead of K1 + K3, and the result equals the oracle bit for bit."""
    cfg = synth.CONFIGS[0]
    pb = synth.packed_batch(cfg, range(4))
    eng = vg.GridEngine()
    monkeypatch.delenv("VG_SMALL", raising=False)
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g, st = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec_of(cfg), engine=eng)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    assert any("vg_small_kernel" in n for n in names)
    assert not any("vg_tables" in n or "vg_slab" in n for n in names)
    ref, rs = orc.batch(pb.offsets, pb.channels, pb.xyz, geom_of(cfg), workers=orc.host_cores())
    assert_bitwise(g.cpu().numpy(), ref, "cfg0 K13")
    assert [int(v) for v in st[:, 1].cpu()] == [r["nonzero_voxels"] for r in rs]


def test_pipeline_varying_batch_sizes_without_syncs():
    """Consecutive submissions of different sizes (every slot reallocates its
    output, counters, inputs and workspace) queued with no host sync: each
    result equals the serial path. Pipeline-owned buffers are registered with
    the pipeline's streams, so a dropped buffer is not reused while an earlier
    batch's kernels may still touch it."""
    from paper_2211_08506_b200.loader import GridPipeline

    cfg = synth.CONFIGS[0]
    spec = spec_of(cfg)
    pipe = GridPipeline(spec, depth=2)
    sizes = [3, 40, 7, 64, 1, 33, 64, 2, 50, 9]
    batches, results = [], []
    start = 0
    for n in sizes:
        pb = synth.packed_batch(cfg, range(start, start + n))
        start += n
        batches.append(pb)
        r = pipe.submit(pb.offsets, pb.channels, pb.xyz)
        # keep a device copy of each result, ordered after its batch
        torch.cuda.current_stream().wait_event(r.ready)
        results.append((r.grids.clone(), r.stats.clone()))
    torch.cuda.synchronize()
    for pb, (g, st) in zip(batches, results):
        g_ref, s_ref = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
        assert_bitwise(g.cpu().numpy(), g_ref.cpu().numpy(), "varying sizes")
        assert np.array_equal(st.cpu().numpy(), s_ref.cpu().numpy())


def test_pipeline_per_slot_compute_streams():
    """Every slot runs its K3 on its own compute stream (the next batch's K3
    starts in the previous one's tail). Same-size batches queued back to back,
    each consumed on the caller's stream and released to the pipeline by an
    event: every result equals the serial path. Submissions that rewrite the
    same caller buffer stay ordered: the buffer ends with the last batch."""
    from paper_2211_08506_b200.loader import GridPipeline

    cfg = synth.CONFIGS[0]
    spec = spec_of(cfg)
    for depth in (2, 3):
        pipe = GridPipeline(spec, depth=depth)
        assert len(pipe.compute_streams) == depth
        cur = torch.cuda.current_stream()
        batches, results, released = [], [], []
        for k in range(7):
            pb = synth.packed_batch(cfg, range(100 * k, 100 * k + 48))
            batches.append(pb)
            rel = released[k - depth] if k >= depth else None   # consumer of the reused slot
            r = pipe.submit(pb.offsets, pb.channels, pb.xyz, release=rel)
            cur.wait_event(r.ready)
            results.append((r.grids.clone(), r.stats.clone()))
            ev = torch.cuda.Event()
            ev.record(cur)
            released.append(ev)
        done = torch.cuda.Event()
        done.record(pipe.join())
        done.synchronize()
        torch.cuda.synchronize()
        for pb, (g, st) in zip(batches, results):
            g_ref, s_ref = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
            assert_bitwise(g.cpu().numpy(), g_ref.cpu().numpy(), f"depth {depth}")
            assert np.array_equal(st.cpu().numpy(), s_ref.cpu().numpy())
    # the same caller buffer written by consecutive submissions (different
    # compute streams): the writes stay in submission order
    pipe = GridPipeline(spec, depth=2)
    out = torch.empty((48, cfg.channels, *cfg.shape), dtype=torch.float32, device="cuda")
    st = torch.empty((48, 2), dtype=torch.int64, device="cuda")
    pipe.order_after(torch.cuda.current_stream())
    last = None
    for k in range(6):
        pb = synth.packed_batch(cfg, range(100 * k, 100 * k + 48))
        last = pipe.submit(pb.offsets, pb.channels, pb.xyz, out=out, stats=st)
    last.ready.synchronize()
    g_ref, s_ref = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
    assert_bitwise(out.cpu().numpy(), g_ref.cpu().numpy(), "same out, last batch")
    assert np.array_equal(st.cpu().numpy(), s_ref.cpu().numpy())


def test_pipeline_edge_batches():
    """GridPipeline over an empty batch, a batch of empty molecules and a
    periodic spec, reusing slots: every result equals the serial path and the
    library reports the kernels it launched."""
    from paper_2211_08506_b200.loader import GridPipeline

    cfg = synth.CONFIGS[0]
    spec = spec_of(cfg)
    pipe = GridPipeline(spec, depth=2)
    r0 = pipe.submit(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros((0, 3)))
    r0.ready.synchronize()
    assert tuple(r0.grids.shape) == (0, 5, 32, 32, 32) and pipe.launches == 0
    r1 = pipe.submit(np.zeros(4, np.int64), np.zeros(0, np.int32), np.zeros((0, 3)))
    r1.ready.synchronize()
    assert not r1.grids.any() and pipe.launches == 1          # one kernel, no tables
    pb = synth.packed_batch(cfg, range(5))
    r2 = pipe.submit(pb.offsets, pb.channels, pb.xyz)
    r2.ready.synchronize()
    g_ref, _ = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
    assert_bitwise(r2.grids.cpu().numpy(), g_ref.cpu().numpy(), "pipeline after empty")
    assert pipe.launches == 2                                 # small batch: K13 alone
    cell = vg.LatticeCell((10.0, 10.0, 10.0))
    pspec = vg.GridSpec((32, 32, 32), 5, vg.BoundingBox((0, 0, 0), (10, 10, 10)), 0.5, cell)
    ppipe = GridPipeline(pspec)
    r3 = ppipe.submit(pb.offsets, pb.channels, np.mod(pb.xyz, 10.0))
    r3.ready.synchronize()
    g_per, _ = vg.generate_packed(pb.offsets, pb.channels, np.mod(pb.xyz, 10.0), pspec)
    assert_bitwise(r3.grids.cpu().numpy(), g_per.cpu().numpy(), "pipeline periodic")


def test_pipeline_binned_batches_k2_on_tables_stream():
    """Large molecules through GridPipeline: K2 (bins) runs on the tables
    stream next to K1, K3 reads the bins on the compute stream; bits equal the
    serial path across slot reuse."""
    from paper_2211_08506_b200.loader import GridPipeline, pinned_csr

    cfg = synth.CONFIGS[3]
    spec = spec_of(cfg)
    pipe = GridPipeline(spec, depth=2)
    batches = [synth.packed_batch(cfg, [i, i + 1]) for i in (0, 4, 9)]
    for pb in batches:
        before = pipe.launches
        res = pipe.submit(*pinned_csr(pb.offsets, pb.channels, pb.xyz))
        res.ready.synchronize()
        assert pipe.launches - before == 3          # K1, K2, K3
        g_ref, s_ref = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec)
        assert_bitwise(res.grids.cpu().numpy(), g_ref.cpu().numpy(), "binned pipeline")
        assert np.array_equal(res.stats.cpu().numpy(), s_ref.cpu().numpy())


def test_unaligned_output_pointer_vs_oracle():
    """An output view whose data pointer is not 16-byte aligned takes the
    scalar-slot kernels (no 128-bit stores), binned and fused paths alike."""
    for k, idx in ((0, range(6)), (3, [2])):
        cfg = synth.CONFIGS[k]
        pb = synth.packed_batch(cfg, idx)
        B = pb.n_molecules
        H, W, D = cfg.shape
        n = B * cfg.channels * H * W * D
        buf = torch.full((n + 1,), 7.0, device="cuda")
        out = buf[1:].view(B, cfg.channels, H, W, D)
        assert out.data_ptr() % 16 != 0
        vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec_of(cfg), out=out)
        ref, _ = orc.batch(pb.offsets, pb.channels, pb.xyz, geom_of(cfg), workers=orc.host_cores())
        assert_bitwise(out.cpu().numpy(), ref, f"unaligned cfg{k}")
        assert float(buf[0]) == 7.0


@pytest.mark.parametrize("env", [{"VG_WS": "1", "VG_WS_NP": "1"},
                                 {"VG_WS": "1", "VG_WS_NP": "2", "VG_WS_STAGES": "5"},
                                 {"VG_WS": "1", "VG_WS_NP": "1", "VG_WS_CAP": "8",
                                  "VG_WS_STAGES": "2"},
                                 {"VG_WS": "1", "VG_WS_NP": "2", "VG_WS_M": "2"}])
def test_warp_specialised_k3w_vs_oracle(env, monkeypatch):
    """The persistent, warp-specialised K3W (producer warps, mbarrier ring,
    cp.async.bulk staging; opt-in with VG_WS=1) gives the oracle's bits and
    counters on binned batches: cfg3 clusters, a tiny staging capacity that
    forces segments, and mixed molecule sizes with an invalid atom."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = synth.CONFIGS[3]
    _compare_with_oracle(cfg, [0, 5, 17])
    rng = np.random.default_rng(23)
    sizes = [1300, 0, 5, 2100, 800]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ch = rng.integers(0, 3, size=off[-1]).astype(np.int32)
    xyz = rng.normal(6.0, 2.5, size=(off[-1], 3))
    spec = vg.GridSpec((38, 30, 48), 3, vg.BoundingBox((0, 0, 0), (12, 12, 12)), 0.45)
    geom = orc.Geometry((38, 30, 48), 3, (0, 0, 0), (12, 12, 12), 0.45)
    g, st = vg.generate_packed(off, ch, xyz, spec)
    ref, rs = orc.batch(off, ch, xyz, geom, workers=orc.host_cores())
    assert_bitwise(g.cpu().numpy(), ref, f"K3W mixed {env}")
    s = st.cpu().numpy()
    assert [int(v) for v in s[:, 0]] == [r["voxel_writes"] for r in rs]
    assert [int(v) for v in s[:, 1]] == [r["nonzero_voxels"] for r in rs]
