"""Input validation and stream/device safety of the sm_100a path.

* The reference raises ValueError for a channel outside [0, C) or a
  non-finite position (gridgen.py:86-90, 114-119; core.py:190-199): host
  inputs are checked before the launch, device inputs by K1, which flags the
  molecule (voxel_writes < 0) and never splats the atom — on the binned (K2)
  path too, where a bad channel used to index past the bin counters.
* GridPipeline orders its streams after the caller's current stream
  (device inputs produced or converted there, no sync before submit).
* Kernel attributes are configured once per device before any launch, also
  when 8 host threads make the first launch together.
"""

from __future__ import annotations

import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

from _golden import assert_bitwise
from oracle import voxgrid_oracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2211_08506_b200 as vg  # noqa: E402
from paper_2211_08506_b200 import synth  # noqa: E402
from paper_2211_08506_b200.loader import GridPipeline, pinned_csr  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def spec_of(cfg):
    return vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                       cfg.sigma)


def geom_of(cfg):
    return orc.Geometry(cfg.shape, cfg.channels, cfg.box_origin, cfg.box_extents, cfg.sigma)


def _corrupt(pb, kind, atom):
    ch, xyz = pb.channels.copy(), pb.xyz.copy().reshape(-1, 3)
    if kind == "channel_high":
        ch[atom] = 1000
    elif kind == "channel_C":
        ch[atom] = int(ch.max()) + 100
    elif kind == "channel_neg":
        ch[atom] = -3
    elif kind == "nan":
        xyz[atom, 1] = np.nan
    elif kind == "inf":
        xyz[atom, 2] = -np.inf
    return ch, xyz


KINDS = ["channel_high", "channel_neg", "nan", "inf"]


@pytest.mark.parametrize("kind", KINDS)
def test_host_inputs_raise_before_launch(kind):
    cfg = synth.CONFIGS[0]
    pb = synth.packed_batch(cfg, range(6))
    atom = int(pb.offsets[3]) + 2
    ch, xyz = _corrupt(pb, kind, atom)
    with pytest.raises(ValueError, match="molecule 3"):
        vg.generate_packed(pb.offsets, ch, xyz, spec_of(cfg))
    pipe = GridPipeline(spec_of(cfg))
    with pytest.raises(ValueError, match="molecule 3"):
        pipe.submit(*pinned_csr(pb.offsets, ch, xyz))


def _expected_without(cfg, pb, atom):
    """Grids of the batch with `atom` removed (what the kernel computes for a
    flagged molecule) from the oracle."""
    keep = np.ones(len(pb.channels), dtype=bool)
    keep[atom] = False
    counts = np.diff(pb.offsets)
    b = int(np.searchsorted(pb.offsets, atom, side="right") - 1)
    counts[b] -= 1
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return orc.batch(off, pb.channels[keep], pb.xyz.reshape(-1, 3)[keep], geom_of(cfg),
                     workers=orc.host_cores()), b


@pytest.mark.parametrize("cfg_i,kind", [(0, k) for k in KINDS] + [(3, "channel_C"),
                                                                  (3, "channel_high"),
                                                                  (3, "nan"), (4, "channel_neg")])
def test_device_inputs_flagged_and_never_splatted(cfg_i, kind):
    cfg = synth.CONFIGS[cfg_i]
    idx = range(3) if cfg_i == 3 else range(8)
    pb = synth.packed_batch(cfg, idx)
    atom = int(pb.offsets[1]) + 5
    ch, xyz = _corrupt(pb, kind, atom)
    off_d = torch.from_numpy(pb.offsets).cuda()
    ch_d = torch.from_numpy(ch).cuda()
    xyz_d = torch.from_numpy(xyz).cuda()
    with pytest.raises(ValueError, match=r"molecules \[1\]"):
        vg.generate_packed(off_d, ch_d, xyz_d, spec_of(cfg))
    guard = 7.5
    B = pb.n_molecules
    H, W, D = cfg.shape
    buf = torch.full((B * cfg.channels * H * W * D + 64,), guard, device="cuda")
    out = buf[:-64].view(B, cfg.channels, H, W, D)
    grids, stats = vg.generate_packed(off_d, ch_d, xyz_d, spec_of(cfg), out=out, check=False)
    st = stats.cpu().numpy()
    assert list(vg.flagged_molecules(stats)) == [1]
    (ref, ref_stats), b = _expected_without(cfg, pb, atom)
    assert b == 1
    assert_bitwise(grids.cpu().numpy(), ref, f"flagged cfg{cfg_i} {kind}")
    assert int(st[1, 0]) & ((1 << 63) - 1) == ref_stats[1]["voxel_writes"]
    assert [int(v) for v in st[:, 1]] == [r["nonzero_voxels"] for r in ref_stats]
    assert [int(v) for i, v in enumerate(st[:, 0]) if i != 1] == \
        [r["voxel_writes"] for i, r in enumerate(ref_stats) if i != 1]
    assert bool((buf[-64:] == guard).all())


def test_pipeline_device_inputs_flagged():
    cfg = synth.CONFIGS[0]
    pb = synth.packed_batch(cfg, range(5))
    ch, xyz = _corrupt(pb, "channel_high", int(pb.offsets[2]))
    pipe = GridPipeline(spec_of(cfg))
    res = pipe.submit(torch.from_numpy(pb.offsets).cuda(), torch.from_numpy(ch).cuda(),
                      torch.from_numpy(xyz).cuda())
    with pytest.raises(ValueError, match=r"molecules \[2\]"):
        res.check()
    ok = pipe.submit(*[torch.from_numpy(a).cuda() for a in (pb.offsets, pb.channels, pb.xyz)])
    ok.check()


def test_pipeline_orders_after_current_stream_producer():
    """Inputs produced on the caller's stream after a long kernel, in dtypes
    the pipeline converts (int64 channels, float32 xyz), submitted with no
    synchronisation: the pipeline's copy/tables/compute streams must wait."""
    cfg = synth.CONFIGS[4]
    pb = synth.packed_batch(cfg, range(40))
    xyz32 = pb.xyz.astype(np.float32)
    spec = spec_of(cfg)
    ref, ref_st = vg.generate_packed(pb.offsets, pb.channels, xyz32.astype(np.float64), spec)
    ref = ref.cpu().numpy()
    pipe = GridPipeline(spec)
    ch_src = torch.from_numpy(pb.channels.astype(np.int64)).cuda()
    xyz_src = torch.from_numpy(xyz32).cuda()
    off_src = torch.from_numpy(pb.offsets).cuda()
    big = torch.randn(6144, 6144, device="cuda")
    torch.cuda.synchronize()
    for rnd in range(3):
        slow = big @ big                       # ~ms on the current stream
        zero = (slow[0, 0] * 0).to(torch.int64)
        ch = ch_src + zero                     # int64, produced after the matmul
        xyz = xyz_src + zero.to(torch.float32)  # float32, produced after the matmul
        res = pipe.submit(off_src, ch, xyz)
        del ch, xyz                            # the pipeline keeps what it needs alive
        res.ready.synchronize()
        assert_bitwise(res.grids.cpu().numpy(), ref, f"producer ordering round {rnd}")
        assert np.array_equal(res.stats.cpu().numpy(), ref_st.cpu().numpy())


def test_first_launch_from_eight_threads_large_smem():
    """Fresh process: 8 host threads make the first K3 launch of a cfg3-shaped
    batch (K2 and K3 need > 48 KB of dynamic shared memory) at the same time;
    every launch succeeds and gives the serial bits."""
    code = textwrap.dedent(f"""
        import sys, threading
        sys.path.insert(0, {str(ROOT)!r})
        import numpy as np, torch
        import paper_2211_08506_b200 as vg
        from paper_2211_08506_b200 import synth
        cfg = synth.CONFIGS[3]
        pb = synth.packed_batch(cfg, [0])
        spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                           cfg.sigma)
        torch.cuda.init()
        start = threading.Barrier(8)
        outs, errs = [None] * 8, []
        def work(i):
            try:
                torch.cuda.set_device(0)
                eng = vg.GridEngine("cuda:0")
                s = torch.cuda.Stream()
                args = [torch.from_numpy(a).cuda() for a in (pb.offsets, pb.channels, pb.xyz)]
                torch.cuda.synchronize()
                start.wait()
                with torch.cuda.stream(s):
                    g, st = vg.generate_packed(*args, spec, engine=eng, stream=s, check=False)
                s.synchronize()
                outs[i] = (g.cpu().numpy().view(np.uint32), st.cpu().numpy())
            except Exception as exc:
                errs.append(repr(exc))
        th = [threading.Thread(target=work, args=(i,)) for i in range(8)]
        [t.start() for t in th]
        [t.join() for t in th]
        assert not errs, errs
        for g, st in outs[1:]:
            assert np.array_equal(g, outs[0][0]) and np.array_equal(st, outs[0][1])
        print("ok")
    """)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stderr[-3000:]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_launches_follow_the_output_device():
    cfg = synth.CONFIGS[0]
    pb = synth.packed_batch(cfg, range(4))
    ref, _ = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec_of(cfg), device="cuda:0")
    with torch.cuda.device(0):
        g, _ = vg.generate_packed(pb.offsets, pb.channels, pb.xyz, spec_of(cfg), device="cuda:1")
        pipe = GridPipeline(spec_of(cfg), device="cuda:1")
        res = pipe.submit(*pinned_csr(pb.offsets, pb.channels, pb.xyz))
        res.ready.synchronize()
    assert_bitwise(g.cpu().numpy(), ref.cpu().numpy(), "cuda:1")
    assert_bitwise(res.grids.cpu().numpy(), ref.cpu().numpy(), "pipeline cuda:1")


def test_bench_gpus2_runs_two_ranks_with_kernels():
    """`bench.py --gpus 2` with kernels: the script spawns two ranks (sharing
    cuda:0 on a one-GPU box: gloo carries the barrier and the max over ranks),
    each generates its half of the batch, and rank 0 prints one line with the
    whole job's rate, the contract's keys and both ranks' shares."""
    import json
    import os

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    res = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--config", "0",
                          "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 64
    assert [r["molecules"] for r in line["per_rank"]] == [32, 32] or \
        sum(r["molecules"] for r in line["per_rank"]) == 64
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    for key in ("roofline", "clocks", "ms_per_step", "higher_is_better"):
        assert key in line
