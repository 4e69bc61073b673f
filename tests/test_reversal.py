"""Grid reversal against the reference.

Peaks are exact (CPU, golden from the reference); loss / gradient /
descent run on the GPU and match the reference within tolerance (fp64 sum
order and float32 expm1 ulps may steer the descent slightly), plus the
reference test suite's own properties (test_reversal.py)."""

from __future__ import annotations

import json
import warnings

import numpy as np
import pytest

import paper_2211_08506_b200 as vg
from _golden import GOLDEN
from paper_2211_08506_b200 import reversal as rv

REV = json.loads((GOLDEN / "reversal.json").read_text())
SPEC = vg.GridSpec((24, 24, 24), 2, vg.BoundingBox((0, 0, 0), (12, 12, 12)), 0.5)


class _HostGrid:
    """Grid stand-in over a host array (peak detection needs no GPU)."""

    def __init__(self, spec, data):
        self.spec, self.data = spec, data


@pytest.mark.parametrize("i", range(len(REV["random_peaks"])))
def test_peaks_match_reference_on_random_grids(i):
    rec = REV["random_peaks"][i]
    spec = vg.GridSpec((8, 8, 8), 1, vg.BoundingBox((0, 0, 0), (1, 1, 1)), 0.1)
    data = np.array(rec["data"], dtype=np.float32).reshape(1, 8, 8, 8)
    got = rv.detect_peaks(_HostGrid(spec, data), rec["threshold"])
    assert [[p.channel, list(p.index), p.value, p.persistence] for p in got] == rec["peaks"]


def test_config_validation():
    for kw in ({"learning_rate": 0}, {"tolerance": 0}, {"max_iters": 0},
               {"persistence_threshold": 1.0}):
        with pytest.raises(ValueError):
            vg.ReversalConfig(**kw)
    with pytest.raises(ValueError):
        rv.detect_peaks(_HostGrid(SPEC, -np.ones((2, 24, 24, 24), np.float32)))
    assert len(rv.detect_peaks(_HostGrid(SPEC, np.zeros((2, 24, 24, 24), np.float32)))) == 0


def _grid(chans, pos):
    g, _ = vg.generate_grid(vg.ParticleSet(np.array(chans), np.array(pos)), SPEC)
    return g


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(REV["cases"])))
def test_reversal_matches_reference(i):
    rec = REV["cases"][i]
    grid = _grid(rec["chans"], rec["pos"])
    peaks = vg.detect_peaks(grid)
    assert [[p.channel, list(p.index), p.value, p.persistence, list(p.seed)]
            for p in peaks] == rec["peaks"]
    st = vg.ReversalState(np.array(rec["chans"]), np.array(rec["cand"]))
    assert vg.loss(grid, st) == pytest.approx(rec["loss"], rel=1e-12)
    np.testing.assert_allclose(vg.loss_gradient(grid, st), np.array(rec["grad"]),
                               rtol=1e-5, atol=1e-12)
    ref = rec["refined"]
    state = vg.refine_coords(grid, st)
    np.testing.assert_allclose(state.positions, np.array(ref["pos"]), atol=2e-5)
    assert state.loss < max(10 * ref["loss"], 1e-11)
    assert state.converged == ref["converged"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        parts = vg.reverse_grid(grid)
    rows = parts.to_rows()
    exp = np.array(rec["reversed"]).reshape(-1, 4)
    assert rows.shape == exp.shape
    np.testing.assert_array_equal(rows[:, 0], exp[:, 0])
    np.testing.assert_allclose(rows[:, 1:], exp[:, 1:], atol=2e-5)


@pytest.mark.gpu
def test_reference_reversal_properties():
    # reference test_reversal.py:149-181, 222-229, 266-304
    pts = [[4.0, 5.0, 6.0], [8.0, 7.0, 5.5]]
    grid = _grid([0, 1], pts)
    truth = vg.ReversalState(np.array([0, 1]), np.array(pts))
    assert vg.loss(grid, truth) < 1e-10
    moved = vg.ReversalState(np.array([0, 1]), np.array(pts) + [0.5, 0, 0])
    assert vg.loss(grid, moved) > vg.loss(grid, truth)
    one = _grid([0], [[5.0, 6.0, 7.0]])
    assert np.linalg.norm(vg.loss_gradient(one, vg.ReversalState(np.array([0]),
                                                                  np.array([[5.0, 6.0, 7.0]])))) < 1e-6
    st = vg.refine_coords(one, vg.ReversalState(np.array([0]), np.array([[5.0, 6.0, 7.0]])))
    assert st.iterations == 0 and st.converged
    with pytest.raises(ValueError):
        vg.loss(one, vg.ReversalState(np.array([7]), np.array([[6.0, 6.0, 6.0]])))
    with pytest.raises(ValueError):
        vg.refine_coords(one, vg.ReversalState(np.zeros(0, int), np.zeros((0, 3))))
    zero = vg.Grid(SPEC, grid.data * 0)
    assert len(vg.reverse_grid(zero)) == 0
    with pytest.warns(vg.CountMismatchWarning):
        vg.reverse_grid(vg.Grid(SPEC, grid.data * 2))
    cell = vg.LatticeCell((12.0, 12.0, 12.0))
    pspec = vg.GridSpec((24, 24, 24), 2, vg.BoundingBox((0, 0, 0), (12, 12, 12)), 0.5, cell)
    with pytest.raises(NotImplementedError):
        vg.reverse_grid(vg.Grid(pspec, grid.data))


@pytest.mark.gpu
def test_gradient_matches_finite_differences():
    # reference test_reversal.py:195-219 (fp32 grids here; fp64 grids are out of scope)
    rng = np.random.default_rng(55)
    spec = vg.GridSpec((16, 16, 16), 2, vg.BoundingBox((0, 0, 0), (8, 8, 8)), 0.45)
    for _ in range(4):
        n = int(rng.integers(1, 4))
        truth = vg.ParticleSet(rng.integers(0, 2, size=n), rng.uniform(2.2, 5.8, size=(n, 3)))
        ref, _ = vg.generate_grid(truth, spec)
        cand = truth.positions + rng.uniform(-0.3, 0.3, size=(n, 3))
        an = vg.loss_gradient(ref, vg.ReversalState(truth.channels.copy(), cand))
        h = 2e-3 * spec.sigma
        for a in range(n):
            for axis in range(3):
                up, dn = cand.copy(), cand.copy()
                up[a, axis] += h
                dn[a, axis] -= h
                fd = (vg.loss(ref, vg.ReversalState(truth.channels.copy(), up))
                      - vg.loss(ref, vg.ReversalState(truth.channels.copy(), dn))) / (2 * h)
                assert abs(fd - an[a, axis]) <= 2e-2 * max(abs(an[a, axis]), 1e-9) + 1e-9


@pytest.mark.gpu
def test_estimator_and_cli_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    clouds = []
    for _ in range(2):
        pts = []
        while len(pts) < 3:
            p = rng.uniform(2.5, 9.5, size=3)
            if all(np.linalg.norm(p - q) >= 3.0 for q in pts):
                pts.append(p)
        clouds.append(np.column_stack([rng.integers(0, 2, size=3), np.array(pts)]))
    est = vg.GaussianVoxelizer(grid_size=24, sigma=0.5, n_channels=2,
                               box=((0, 0, 0), (12, 12, 12))).fit(clouds)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        rec = est.inverse_transform(est.transform(clouds))
    for truth, got in zip(clouds, rec):
        assert got.shape == truth.shape
        for c in (0, 1):
            t, r = truth[truth[:, 0] == c, 1:], got[got[:, 0] == c, 1:]
            assert t.shape == r.shape
            for p in t:
                assert np.min(np.linalg.norm(r - p, axis=1)) < 0.25
    from paper_2211_08506_b200 import cli

    g = est.transform(clouds[:1])[0]
    vg.write_npy(g, tmp_path / "g.npy")
    assert cli.cli_main(["reverse", "--input", str(tmp_path / "g.npy"), "--variance", "0.5",
                         "--box", "0,0,0,12,12,12", "--output", str(tmp_path / "o.csv")]) == 0
    lines = (tmp_path / "o.csv").read_text().strip().splitlines()
    assert len(lines) == 3


@pytest.mark.gpu
@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("max_iters,tol", [(5000, 1e-12), (7, 1e-30), (40, 1e-30)])
def test_device_descent_equals_host_loop(max_iters, tol, graphs, monkeypatch):
    """refine_coords (the loop on the device, stop flag read every few
    iterations) takes exactly the steps of the host-driven loop: same
    iterations, same best loss, bit-identical positions; including stops by
    max_iters in the middle of a queued block."""
    from paper_2211_08506_b200 import reversal as rv

    monkeypatch.setattr(rv, "_USE_GRAPHS", graphs)
    for i in range(min(3, len(REV["cases"]))):
        rec = REV["cases"][i]
        grid = _grid(rec["chans"], rec["pos"])
        seeds = vg.ReversalState(np.array(rec["chans"]), np.array(rec["cand"]))
        conf = vg.ReversalConfig(max_iters=max_iters, tolerance=tol)
        a = rv.refine_coords(grid, seeds, conf)
        b = rv._refine_host(grid, seeds, conf)
        assert a.iterations == b.iterations
        assert a.loss == b.loss
        assert a.converged == b.converged and a.diverged == b.diverged
        assert np.array_equal(a.positions, b.positions)


@pytest.mark.gpu
def test_batched_descent_equals_single_reversals():
    """refine_coords_batch / reverse_grids: every molecule's result equals its
    own refine_coords bit for bit (different atom counts, stops at different
    iterations, a converged seed)."""
    from paper_2211_08506_b200 import reversal as rv

    grids, seeds = [], []
    for i in range(min(4, len(REV["cases"]))):
        rec = REV["cases"][i]
        grids.append(_grid(rec["chans"], rec["pos"]))
        seeds.append(vg.ReversalState(np.array(rec["chans"]), np.array(rec["cand"])))
    exact = [[4.0, 5.0, 6.0], [8.0, 7.0, 5.5]]
    grids.append(_grid([0, 1], exact))
    seeds.append(vg.ReversalState(np.array([0, 1]), np.array(exact)))
    for conf in (vg.ReversalConfig(), vg.ReversalConfig(max_iters=23, tolerance=1e-30)):
        batch = rv.refine_coords_batch(grids, seeds, conf)
        for g, s_, b in zip(grids, seeds, batch):
            a = rv.refine_coords(g, s_, conf)
            assert a.iterations == b.iterations and a.loss == b.loss
            assert a.converged == b.converged and a.diverged == b.diverged
            assert np.array_equal(a.positions, b.positions)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        many = rv.reverse_grids(grids)
        for g, p in zip(grids, many):
            one = rv.reverse_grid(g)
            assert np.array_equal(one.to_rows(), p.to_rows())


def test_batched_reversal_validates_without_gpu():
    """refine_coords_batch rejects mismatched inputs before touching the GPU."""
    from paper_2211_08506_b200 import reversal as rv

    assert rv.refine_coords_batch([], []) == []
    import torch

    g1 = vg.Grid(SPEC, torch.zeros((2,) + SPEC.shape))
    other = vg.GridSpec(SPEC.shape, 2, vg.BoundingBox((0, 0, 0), (6, 6, 6)), 0.5)
    g2 = vg.Grid(other, torch.zeros((2,) + SPEC.shape))
    seeds = vg.ReversalState(np.array([0]), np.array([[1.0, 1.0, 1.0]]))
    with pytest.raises(ValueError):
        rv.refine_coords_batch([g1], [seeds, seeds])
    with pytest.raises(ValueError):
        rv.refine_coords_batch([g1, g2], [seeds, seeds])
