"""Randomised parity (hypothesis, 1000 + 250 + 300 derandomised cases): random shapes, channel counts, boxes,
sigmas, thresholds, periodic cells and molecule sizes, GPU path vs the CPU
oracle, bit for bit, with identical GenStats counters. Complements the fixed
cases of test_gpu_parity.py with inputs nobody chose by hand. The outputs sit
inside guard bands that must stay untouched (bounds check in place of
compute-sanitizer, which this GPU pool does not allow)."""

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
    # output inside a guarded buffer: no kernel may write outside its grids
    B = len(sizes)
    n_out = B * C * H * W * D
    guard = 4096
    buf = torch.full((guard + n_out + guard,), -7.0, device="cuda")
    grids = buf[guard:guard + n_out].view(B, C, H, W, D)
    _, st_ = vg.generate_packed(offsets, ch, xyz, spec, threshold=thr, out=grids)
    assert bool((buf[:guard] == -7.0).all()) and bool((buf[guard + n_out:] == -7.0).all())
    geom = orc.Geometry((H, W, D), C, origin, ext, sigma, periodic)
    ref, rs = orc.batch(offsets, ch, xyz, geom, threshold=thr)
    assert_bitwise(grids.cpu().numpy(), ref, f"random case {case}")
    st_h = st_.cpu().numpy()
    assert [int(v) for v in st_h[:, 0]] == [r["voxel_writes"] for r in rs]
    assert [int(v) for v in st_h[:, 1]] == [r["nonzero_voxels"] for r in rs]


@st.composite
def fused_batches(draw):
    H = draw(st.integers(8, 40))
    W = draw(st.integers(1, 40))
    D = draw(st.sampled_from([4, 8, 12, 16, 20, 24, 32, 40, 7, 13]))
    C = draw(st.integers(2, 6))
    ext = tuple(draw(st.floats(2.0, 12.0)) for _ in range(3))
    sigma = draw(st.floats(0.1, 1.0))
    thr = draw(st.one_of(st.none(), st.floats(1e-7, 0.05)))
    sizes = draw(st.lists(st.integers(0, 90), min_size=4, max_size=14))
    seed = draw(st.integers(0, 2**31 - 1))
    bulk = draw(st.booleans())
    return H, W, D, C, ext, sigma, thr, sizes, seed, bulk


@settings(max_examples=250, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow])
@given(fused_batches())
def test_random_fused_batches_with_tapered_tail_match_oracle(case):
    """The two-kernel path (VG_SMALL=0) with the launch's tapered tail forced
    (VG_TAPER=2: the last third of the molecules in quarter-length y-chunks;
    VG_TASK_KB keeps long chunks to divide) on random shapes, with bulk-copy or
    cp.async staging: bit-exact vs the oracle, counters identical, nothing
    written outside the grids."""
    import os

    H, W, D, C, ext, sigma, thr, sizes, seed, bulk = case
    origin = (0.0, 0.0, 0.0)
    rng = np.random.default_rng(seed)
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n = int(offsets[-1])
    xyz = rng.uniform(-1.0, np.array(ext) + 1.0, (n, 3))
    ch = rng.integers(0, C, n).astype(np.int32)
    spec = vg.GridSpec((H, W, D), C, vg.BoundingBox(origin, ext), sigma)
    B = len(sizes)
    n_out = B * C * H * W * D
    guard = 4096
    buf = torch.full((guard + n_out + guard,), -7.0, device="cuda")
    grids = buf[guard:guard + n_out].view(B, C, H, W, D)
    hooks = {"VG_SMALL": "0", "VG_TAPER": "2", "VG_TASK_KB": "4096", "VG_FUSE": "1",
             "VG_BULK": "1" if bulk else "0"}
    old = {k: os.environ.get(k) for k in hooks}
    os.environ.update(hooks)
    try:
        _, st_ = vg.generate_packed(offsets, ch, xyz, spec, threshold=thr, out=grids)
        torch.cuda.synchronize()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert bool((buf[:guard] == -7.0).all()) and bool((buf[guard + n_out:] == -7.0).all())
    geom = orc.Geometry((H, W, D), C, origin, ext, sigma, False)
    ref, rs = orc.batch(offsets, ch, xyz, geom, threshold=thr)
    assert_bitwise(grids.cpu().numpy(), ref, f"tapered case {case}")
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


@pytest.mark.parametrize("k", [0, 3, 4])
def test_workspace_and_stats_stay_in_bounds(k):
    """Through the C-ABI: the workspace (tables, supports, K2 bins) and the
    stats buffer sit between guard bands; vg_generate_f32 writes only inside."""
    from paper_2211_08506_b200 import _native, synth

    cfg = synth.CONFIGS[k]
    pb = synth.packed_batch(cfg, range(3))
    spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                       cfg.sigma)
    eng = vg.GridEngine()
    off = torch.from_numpy(pb.offsets).cuda()
    ch = torch.from_numpy(pb.channels).cuda()
    xyz = torch.from_numpy(pb.xyz).cuda()
    desc = eng.describe(off, ch, xyz.view(-1, 3), spec)
    layout = _native.VgWsLayout()
    lib = _native.lib()
    assert lib.vg_workspace_layout(desc, layout) == 0
    g = 1 << 16
    wsbuf = torch.full((g + layout.total + g,), 0xA5, dtype=torch.uint8, device="cuda")
    stbuf = torch.full((2 * 64 + 2 * 3 + 2 * 64,), -3, dtype=torch.int64, device="cuda")
    out = torch.empty((3, cfg.channels) + tuple(cfg.shape), device="cuda")
    ws_ptr = wsbuf.data_ptr() + g
    st_ptr = stbuf.data_ptr() + 2 * 64 * 8
    rc = lib.vg_generate_f32(desc, out.data_ptr(), ws_ptr, layout.total, st_ptr,
                             torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    assert bool((wsbuf[:g] == 0xA5).all()) and bool((wsbuf[g + layout.total:] == 0xA5).all())
    assert bool((stbuf[:128] == -3).all()) and bool((stbuf[128 + 6:] == -3).all())
    ref, rs = orc.batch(pb.offsets, pb.channels, pb.xyz,
                        orc.Geometry(cfg.shape, cfg.channels, cfg.box_origin, cfg.box_extents,
                                     cfg.sigma), workers=orc.host_cores())
    assert_bitwise(out.cpu().numpy(), ref, f"guarded cfg{k}")
    st = stbuf[128:134].view(3, 2).cpu().numpy()
    assert [int(v) for v in st[:, 1]] == [r["nonzero_voxels"] for r in rs]
    # a workspace that is not 16-byte aligned is refused (the table rows are
    # staged with 16-byte copies), before anything is launched
    rc = lib.vg_generate_f32(desc, out.data_ptr(), ws_ptr + 4, layout.total, st_ptr,
                             torch.cuda.current_stream().cuda_stream)
    assert rc == _native.VG_ERR_INVALID and b"16-byte" in lib.vg_last_error()
