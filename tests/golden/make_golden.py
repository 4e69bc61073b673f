"""Generate the golden fixtures from the REAL reference implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``voxgrid`` read-only from
``$VOXGRID_REF`` (default /root/reference/pkg/src) and writes, under
tests/golden/:

  erf.npz        erf_approx(t, float32) at 60k+ arguments (kernels.py:59-70)
  tables.npz     fused_axis_tables values/supports for random axis cases
                 (kernels.py:217-274), open, thresholded and periodic
  grids.npz      full (C,H,W,D) grids + GenStats from generate_grid
                 (gridgen.py:130-153) for the reference's own KAT-style cases
  configs.json   per-grid sha256 of the float32 bytes + GenStats of
                 generate_batch over samples of BASELINE configs 0-4, the
                 per-molecule-bbox policy and GaussianVoxelizer.transform

The GPU path and the oracle are both checked against these bits. Nothing at
run time on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, os.environ.get("VOXGRID_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(ROOT))

import voxgrid  # noqa: E402  (the reference)
from voxgrid import (  # noqa: E402
    BoundingBox, GridSpec, LatticeCell, ParticleSet, generate_batch, generate_grid)
from voxgrid.kernels import erf_approx, fused_axis_tables  # noqa: E402

from paper_2211_08506_b200 import synth  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def packed_sha(pb) -> str:
    h = hashlib.sha256()
    for arr in (pb.offsets.astype(np.int64), pb.channels.astype(np.int32),
                pb.xyz.astype(np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def make_erf():
    rng = np.random.default_rng(7)
    t = np.concatenate([
        np.linspace(-6, 6, 20001),
        rng.normal(0, 2.5, 20000),
        rng.uniform(-0.6, 0.6, 20000),
        [0.0, -0.0, 5.0, -5.0, 6.0, 9.0, 1e-8, -1e-8, 1e-30, 0.5, 3.0, 30.0, 1e20],
    ]).astype(np.float32)
    e = erf_approx(t, np.float32)
    np.savez_compressed(HERE / "erf.npz", t=t, e=e)


def make_tables():
    rng = np.random.default_rng(11)
    rows = []
    for case in range(60):
        sigma = float(rng.uniform(0.05, 1.5))
        delta = sigma * float(rng.uniform(0.1, 2.5))
        n = int(rng.integers(1, 80))
        origin = float(rng.uniform(-5, 5))
        periodic = case % 4 == 3
        mus = [origin + float(rng.uniform(-0.3, 1.3)) * n * delta for _ in range(3)]
        threshold = float(10 ** rng.uniform(-7, -2)) if case % 5 == 2 else None
        params = [(n, origin, delta), (max(1, n // 2), origin + 0.5, delta * 1.1),
                  (n + 3, origin - 0.25, delta * 0.9)]
        if periodic:
            sigma = min(sigma, 0.9 * min(pn * pd for pn, _, pd in params) / 6.0)
        tabs = fused_axis_tables(mus, params, sigma, np.float32, threshold, periodic)
        rows.append(dict(sigma=sigma, periodic=periodic, threshold=threshold, mus=mus,
                         params=params,
                         values=[t.values.astype(np.float32) for t in tabs],
                         supports=[list(t.support) for t in tabs]))
    flat = {}
    meta = []
    for r_i, r in enumerate(rows):
        for a in range(3):
            flat[f"v{r_i}_{a}"] = r["values"][a]
        meta.append({k: r[k] for k in ("sigma", "periodic", "threshold", "mus", "params",
                                       "supports")})
    np.savez_compressed(HERE / "tables.npz", meta=json.dumps(meta), **flat)


def _grid_case(name, shape, channels, origin, extents, sigma, chans, pos, periodic=None,
               mode="sparse", threshold=None):
    lattice = LatticeCell(tuple(periodic)) if periodic is not None else None
    spec = GridSpec(tuple(shape), channels, BoundingBox(tuple(origin), tuple(extents)), sigma,
                    lattice)
    ps = ParticleSet(np.asarray(chans, dtype=np.int64), np.asarray(pos, dtype=np.float64).reshape(-1, 3),
                     lattice)
    g, st = generate_grid(ps, spec, mode=mode, threshold=threshold)
    return dict(name=name, shape=list(shape), channels=channels, origin=list(origin),
                extents=list(extents), sigma=sigma, periodic=list(periodic) if periodic else None,
                mode=mode, threshold=threshold,
                chans=ps.channels.tolist(), pos=ps.positions.tolist(),
                voxel_writes=st.voxel_writes, erf_evals=st.erf_evals,
                nonzero_voxels=st.nonzero_voxels), g.data


def make_grids():
    cases = []
    rng = np.random.default_rng(2)
    # layout KAT (reference test_core.py:131-142)
    cases.append(_grid_case("layout_kat", (2, 3, 4), 1, (0, 0, 0), (3, 2, 4), 0.08, [0],
                            [[2.5, 0.5, 3.5]]))
    # octants (test_gridgen.py:26-30)
    cases.append(_grid_case("octants", (2, 2, 2), 1, (0, 0, 0), (1, 1, 1), 0.05, [0],
                            [[0.5, 0.5, 0.5]]))
    # anisotropic naive-loop case (test_gridgen.py:71-80): 5 atoms, dense + sparse
    pos = rng.uniform([-1, 0, 2], [2, 4, 4.5], size=(5, 3))
    for mode in ("sparse", "dense"):
        cases.append(_grid_case(f"naive_765_{mode}", (7, 6, 5), 1, (-1, 0, 2), (3, 4, 2.5), 0.4,
                                [0] * 5, pos, mode=mode))
    # erf-count geometry (test_gridgen.py:83-88), multi-channel
    cases.append(_grid_case("aniso_10_12_14", (10, 12, 14), 3, (0, 0, 0), (6, 5, 7), 0.5,
                            [0, 2, 2, 1], [[3.0, 2.5, 3.5], [1.0, 1.0, 1.0], [1.2, 1.1, 0.9],
                                           [5.5, 4.9, 6.8]]))
    # threshold (test_gridgen.py:124-137)
    r15 = np.random.default_rng(15)
    pos = r15.uniform(2.0, 6.0, size=(6, 3))
    for mode, thr in (("sparse", 1e-6), ("dense", 1e-6), ("sparse", None), ("sparse", 3e-3)):
        cases.append(_grid_case(f"threshold_{mode}_{thr}", (24, 24, 24), 1, (0, 0, 0), (8, 8, 8),
                                0.5, [0] * 6, pos, mode=mode, threshold=thr))
    # out-of-box (test_gridgen.py:139-144)
    cases.append(_grid_case("out_of_box", (8, 8, 8), 1, (0, 0, 0), (4, 4, 4), 0.3, [0, 0],
                            [[-10.0, 2.0, 2.0], [2.0, 2.0, 2.0]]))
    # empty
    cases.append(_grid_case("empty", (8, 8, 8), 2, (0, 0, 0), (4, 4, 4), 0.3, [],
                            np.zeros((0, 3))))
    # periodic (test_gridgen.py:147-153, test_acceptance.py:211-227)
    cases.append(_grid_case("periodic_corner", (24, 24, 24), 1, (0, 0, 0), (6, 6, 6), 0.4, [0, 0],
                            [[0.0, 0.0, 0.0], [5.9, 3.0, 0.05]], periodic=(6, 6, 6)))
    r44 = np.random.default_rng(44)
    for trial in range(3):
        edge = float(r44.uniform(5.0, 10.0))
        n = int(r44.integers(12, 33))
        sigma = float(r44.uniform(0.05, 0.15)) * edge
        atoms = int(r44.integers(2, 6))
        p = r44.uniform(0, edge, size=(atoms, 3))
        p[0] = (0.0, 0.0, 0.0)
        p[1] = (edge * 0.9999, 0.5 * edge, 1e-6)
        cases.append(_grid_case(f"periodic_rand{trial}", (n, n + 1, n + 2), 2, (0, 0, 0),
                                (edge, edge, edge), sigma, list(r44.integers(0, 2, atoms)), p,
                                periodic=(edge, edge, edge)))
    # non-multiple-of-4 z (scalar store path), tiny and wide sigma
    r9 = np.random.default_rng(9)
    cases.append(_grid_case("odd_z_9_7_5", (9, 7, 5), 2, (-1, -2, 0.5), (4.0, 3.5, 2.5), 0.3,
                            [0, 1, 1, 0], r9.uniform([-1, -2, 0.5], [3, 1.5, 3], size=(4, 3))))
    cases.append(_grid_case("wide_sigma", (12, 12, 12), 1, (0, 0, 0), (4, 4, 4), 2.0, [0, 0],
                            [[2.0, 2.0, 2.0], [0.5, 3.7, 1.1]]))
    cases.append(_grid_case("tiny_sigma", (16, 16, 16), 2, (0, 0, 0), (8, 8, 8), 0.05,
                            [0, 1, 0], [[4.0, 4.0, 4.0], [1.25, 7.5, 3.3], [4.01, 4.02, 3.99]]))
    # translation equivariance (test_gridgen.py:172-182)
    base = np.array([[2.25, 3.5, 4.125], [5.0, 2.75, 6.5]])
    for s_i, shift in enumerate([(0, 0, 0), (1.5, -2.25, 4.0), (0.1, 0.37, -1.234)]):
        cases.append(_grid_case(f"translate{s_i}", (16, 16, 16), 1, shift, (8, 8, 8), 0.5, [0, 0],
                                base + np.asarray(shift)))
    # a config-0 molecule at 32^3 with every sigma of the reference sweep
    ch, xyz = synth.molecule(synth.CONFIGS[0], 5)
    for sigma in (0.05, 0.1, 0.25, 0.5):
        cases.append(_grid_case(f"cfg0_m5_sigma{sigma}", (32, 32, 32), 5, (0, 0, 0),
                                (10, 10, 10), sigma, ch, xyz))
    meta, arrays = [], {}
    for i, (m, g) in enumerate(cases):
        meta.append(m)
        arrays[f"g{i}"] = g
    np.savez_compressed(HERE / "grids.npz", meta=json.dumps(meta), **arrays)
    return len(cases)


def _batch_record(cfg, indices, spec_policy="fixed"):
    pb = synth.packed_batch(cfg, indices)
    spec = GridSpec(cfg.shape, cfg.channels, BoundingBox(cfg.box_origin, cfg.box_extents),
                    cfg.sigma)
    sets = [ParticleSet(pb.channels[pb.offsets[b]:pb.offsets[b + 1]].astype(np.int64),
                        pb.xyz[pb.offsets[b]:pb.offsets[b + 1]]) for b in range(pb.n_molecules)]
    res = generate_batch(sets, spec, spec_policy=spec_policy, parallelism=1)
    assert not res.errors, res.errors
    recs = []
    for (g, st) in res.results:
        recs.append(dict(sha=sha(g.data), voxel_writes=st.voxel_writes, erf_evals=st.erf_evals,
                         nonzero_voxels=st.nonzero_voxels,
                         channel_sums=[float(v) for v in g.channel_sums()],
                         box=[list(g.spec.box.origin), list(g.spec.box.extents)]))
    return dict(config=cfg.index, indices=list(map(int, indices)), spec_policy=spec_policy,
                inputs_sha=packed_sha(pb), grids=recs)


def make_configs():
    out = {"numpy": np.__version__, "voxgrid": voxgrid.__version__, "batches": []}
    C = synth.CONFIGS
    out["batches"].append(_batch_record(C[0], range(64)))
    out["batches"].append(_batch_record(C[1], list(range(8)) + list(range(100, 1024, 131))))
    out["batches"].append(_batch_record(C[2], list(range(0, 65536, 1024))))
    out["batches"].append(_batch_record(C[3], [0, 1]))
    out["batches"].append(_batch_record(C[4], list(range(0, 4096, 64))))
    out["batches"].append(_batch_record(C[0], range(16), spec_policy="per-molecule-bbox"))
    # GaussianVoxelizer (estimator.py:134-151) on config-0 molecules as (n,4) rows
    from voxgrid import GaussianVoxelizer
    clouds = []
    for b in range(6):
        ch, xyz = synth.molecule(C[0], b)
        clouds.append(np.column_stack([ch.astype(np.float64), xyz]))
    est = GaussianVoxelizer(grid_size=24, sigma=0.4).fit(clouds)
    grids = est.transform(clouds)
    per = GaussianVoxelizer(grid_size=(20, 16, 12), sigma=0.5, box="per-sample").fit(clouds)
    grids_per = per.transform(clouds)
    out["estimator"] = dict(
        shared=dict(grid_size=24, sigma=0.4, channels=est.channels_,
                    box=[list(est.box_.origin), list(est.box_.extents)],
                    shas=[sha(g) for g in grids]),
        per_sample=dict(grid_size=[20, 16, 12], sigma=0.5, shas=[sha(g) for g in grids_per]))
    (HERE / "configs.json").write_text(json.dumps(out, indent=1))


IO_XYZ = [
    "1\n\nC 0 0 0\n",
    "3\nwater\nO 0.0 0.0 0.117\nH 0.0 0.757 -0.467\nH 0.0 -0.757 -0.467\n",
    "5\nmethane\nC 0.0 0.0 0.0\nH 0.629 0.629 0.629\nH -0.629 -0.629 0.629\n"
    "H -0.629 0.629 -0.629\nH 0.629 -0.629 -0.629\n",
    "4\nmixed\nFe 1 2 3\n\nZn 1.5 2 3\nS 0 0 -1e-3\nP 4 4 4\n",
    "3\ncomment\nC 0 0 0\nC 1 0 0\n",
    "1\n\nC 0 0 0\nC 1 0 0\n",
    "1\n\nXx 0 0 0\n",
    "1\n\nC 0 zero 0\n",
    "banana\n\nC 0 0 0\n",
    "-2\n\n",
    "",
    "2\n\nC 0 0 0 9\nH 1 1 1\n",
    "1\n\nC nan 0 0\n",
]
IO_CSV = [
    "0,0.5,0.5,0.5\n1,0.0,0.1,0.2\n",
    "channel,x,y,z\n2,1,2,3\n\n0,4,5,6\n",
    "",
    "0,1,2\n",
    "a,1,2,3\n",
    "1,1,2,3\n-1,0,0,0\n",
    "0,1,x,3\n",
    "0,1,inf,3\n",
    '0,"1,2",3\n',
]


def make_io():
    from voxgrid.io import parse_points_csv, parse_xyz
    from voxgrid.cli import cli_main
    from voxgrid.bench import synth_corpus
    import tempfile

    out = {"xyz": [], "csv": [], "cli": [], "corpus": {}}
    for text in IO_XYZ:
        try:
            m = parse_xyz(text)
            out["xyz"].append({"text": text, "symbols": list(m.symbols),
                               "positions": m.positions.tolist(),
                               "auto": m.channel_map("auto"), "n_auto": m.n_channels("auto")})
        except ValueError as exc:
            out["xyz"].append({"text": text, "error": str(exc), "line": getattr(exc, "line", None)})
    for text in IO_CSV:
        try:
            ps = parse_points_csv(text)
            out["csv"].append({"text": text, "rows": ps.to_rows().tolist()})
        except ValueError as exc:
            out["csv"].append({"text": text, "error": str(exc), "line": getattr(exc, "line", None)})
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        (tmp / "water.xyz").write_text(IO_XYZ[1])
        (tmp / "mixed.xyz").write_text(IO_XYZ[3])
        (tmp / "pts.csv").write_text(IO_CSV[0])
        runs = [
            ["--input", "water.xyz", "--grid-size", "24", "--variance", "0.4"],
            ["--input", "water.xyz", "--grid-size", "16,20,12", "--variance", "0.5",
             "--channels", "single", "--mode", "dense"],
            ["--input", "mixed.xyz", "--grid-size", "20", "--variance", "0.3", "--channels", "6",
             "--padding-sigmas", "2.5"],
            ["--input", "pts.csv", "--grid-size", "32", "--variance", "0.05", "--channels", "2",
             "--box", "0,0,0,1,1,1"],
            ["--input", "pts.csv", "--grid-size", "24", "--variance", "0.1", "--periodic",
             "1,1,1"],
        ]
        for args in runs:
            full = ["grid"] + [str(tmp / a) if a.endswith((".xyz", ".csv")) else a for a in args]
            full += ["--output", str(tmp / "o.npy"), "--stats", str(tmp / "s.json")]
            code = cli_main(full)
            rec = {"args": args, "code": code}
            if code == 0:
                arr = np.load(tmp / "o.npy")
                st = json.loads((tmp / "s.json").read_text())
                st.pop("elapsed_ms", None)
                rec.update(sha=sha(arr), shape=list(arr.shape), stats=st)
            out["cli"].append(rec)
    corpus = synth_corpus(7, (8, 40), 48.0, seed=3)
    h = hashlib.sha256()
    for ps in corpus:
        h.update(ps.channels.astype(np.int64).tobytes())
        h.update(ps.positions.astype(np.float64).tobytes())
    out["corpus"] = {"n": 7, "seed": 3, "sha": h.hexdigest()}
    (HERE / "io.json").write_text(json.dumps(out, indent=1))


def make_reversal():
    """Peaks (exact), loss/gradient values and full reversals by the reference."""
    import warnings
    from voxgrid import (ReversalState, detect_peaks, loss, loss_gradient, refine_coords,
                         reverse_grid)

    rng = np.random.default_rng(4242)
    box = BoundingBox((0.0, 0.0, 0.0), (12.0, 12.0, 12.0))
    spec = GridSpec((24, 24, 24), 2, box, 0.5)
    cases = []
    for trial in range(6):
        n = int(rng.integers(1, 7))
        pts = []
        while len(pts) < n:
            p = rng.uniform(2.05, 9.95, size=3)
            if all(np.linalg.norm(p - q) >= 3.0 for q in pts):
                pts.append(p)
        truth = ParticleSet(rng.integers(0, 2, size=n), np.array(pts))
        grid, _ = generate_grid(truth, spec)
        peaks = detect_peaks(grid)
        cand = truth.positions + rng.uniform(-0.3, 0.3, size=(n, 3))
        st = ReversalState(truth.channels.copy(), cand)
        lval = loss(grid, st)
        gval = loss_gradient(grid, st)
        refined = refine_coords(grid, st)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rec = reverse_grid(grid)
        cases.append(dict(
            chans=truth.channels.tolist(), pos=truth.positions.tolist(), cand=cand.tolist(),
            peaks=[[p.channel, list(p.index), p.value, p.persistence, list(p.seed)]
                   for p in peaks],
            loss=lval, grad=gval.tolist(),
            refined=dict(pos=refined.positions.tolist(), loss=refined.loss,
                         iterations=refined.iterations, converged=refined.converged),
            reversed=rec.to_rows().tolist()))
    # peak detection on random (noisy, plateau-rich) grids
    rnd = []
    r2 = np.random.default_rng(123)
    small = GridSpec((8, 8, 8), 1, BoundingBox((0, 0, 0), (1, 1, 1)), 0.1)
    for trial in range(8):
        data = r2.uniform(0.0, 1.0, size=(1, 8, 8, 8)).astype(np.float32)
        if trial % 3 == 0:
            data[data < 0.3] = 0.0
        if trial % 4 == 0:
            data = np.round(data, 1).astype(np.float32)
        thr = float(r2.uniform(0.05, 0.6))
        from voxgrid import Grid as RGrid
        peaks = detect_peaks(RGrid(small, np.ascontiguousarray(data)), thr)
        rnd.append(dict(data=data.ravel().tolist(), threshold=thr,
                        peaks=[[p.channel, list(p.index), p.value, p.persistence] for p in peaks]))
    (HERE / "reversal.json").write_text(json.dumps({"spec": [24, 2, 12.0, 0.5], "cases": cases,
                                                   "random_peaks": rnd}))


if __name__ == "__main__":
    make_reversal()
    make_io()
    make_erf()
    make_tables()
    n = make_grids()
    make_configs()
    print(f"golden fixtures written to {HERE} ({n} grid cases)")
