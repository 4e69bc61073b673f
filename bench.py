#!/usr/bin/env python3
"""Benchmark of the B200 grid-generation hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): 1024 synthetic molecules of the
config-0 distribution -> fp32 grids [1024, 5, 64, 64, 64] over a 12 A cube,
sigma 0.5 (5.37 GB of output per step, 42x the 126 MB L2, so every step
streams to HBM; the atom inputs are tiny and stay resident). ``--config N``
selects another BASELINE config.

A *step* = one pass of the hot path over the batch: K1 (per-atom axis
tables) + K3 (slab gather/store, all voxels incl. zeros, fused nonzero
counters). ``value`` = grids/s over all ranks (inputs resident in HBM);
``e2e`` = the same metric through the public API ``generate_packed`` with
host (pinned) CSR inputs copied H2D and the per-grid stats read back D2H
inside the timed region. ``roofline`` = K3's algorithmic bytes (the output)
per launch / its CUDA-event duration vs the measured HBM peak.

Multi-GPU: one process per GPU. ``--gpus N`` under torchrun uses the
launcher's ranks (WORLD_SIZE must equal N); without a launcher, bench.py
re-executes itself under ``torch.distributed.run`` with N ranks. The
config's fixed batch is split into N cost-balanced contiguous molecule ranges
(strong scaling, the BASELINE "single GPU then sharded over 2/4/8 GPUs";
``--scaling weak`` gives every rank the whole batch size instead). There is
no collective on the data path: NCCL carries only the barrier and the
max-over-ranks time. More ranks than GPUs (plumbing runs on a 1-GPU box)
share devices and switch the timing plumbing to gloo.

``--impl reference`` times the UNMODIFIED reference (``voxgrid`` installed in
baseline/_ref by scripts/install_reference.sh) on this host's cores: a process
pool over the stock ``generate_grid`` on the same batch, plus the
reference's own ``generate_batch(parallelism=ncores)``; the oracle port only
when the install is missing.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", type=int, default=1, help="BASELINE config index (default 1)")
    ap.add_argument("--batch", type=int, default=None, help="molecules per GPU (default: config)")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="strong",
                    help="strong: the config's batch split over the ranks (default); "
                         "weak: every rank processes a full batch of its own")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline budget")
    ap.add_argument("--dist-backend", default="auto",
                    help="timing plumbing backend: auto (nccl, or gloo when ranks share GPUs), "
                         "nccl or gloo")
    ap.add_argument("--dry-run", action="store_true",
                    help="plan shards, synthesize inputs and run the timing plumbing without "
                         "kernels (CPU test of the multi-rank path)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:  # noqa: BLE001
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polling thread)
# ---------------------------------------------------------------------------
_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.period = period_s
        self._stop = threading.Event()
        self._thread = None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # noqa: BLE001
            log(f"[bench] NVML unavailable for clock sampling: {exc}")

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._stop.clear()
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        names = [n for bit, n in _REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# distributed plumbing (barrier + max over ranks only)
# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """Re-execute this script under torch.distributed.run with n ranks (one
    process per GPU); rank 0's JSON line goes to our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    log(f"[bench] --gpus {n} without a launcher: {' '.join(cmd[1:6])} ...")
    return subprocess.call(cmd)


def plan_indices(cfg, B, rank, world, scaling):
    """This rank's molecule indices: a cost-balanced contiguous range of the
    config's batch (strong), or a full batch of its own (weak)."""
    from paper_2211_08506_b200 import shard, synth

    if scaling == "weak":
        return range(rank * B, (rank + 1) * B)
    costs = shard.molecule_costs(synth.atom_counts(cfg, range(B)), cfg.grid_bytes,
                                 shard.BYTES_PER_ATOM)
    return shard.shard_range(B, rank, world, costs)


class Dist:
    """Barrier + max/sum over ranks (timing plumbing only; no data-path
    collective). NCCL on GPUs; gloo on CPU for the multi-process tests."""

    def __init__(self, world, rank, local, backend="nccl"):
        import torch

        self.world, self.rank, self.local = world, rank, local
        self.torch = torch
        self.pg = None
        self.device = "cuda" if backend == "nccl" else "cpu"
        if world > 1:
            import torch.distributed as td

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend == "nccl":
                td.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                td.init_process_group(backend, rank=rank, world_size=world)
            self.td = td
            self.pg = True

    def barrier(self):
        if self.pg:
            self.td.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.device)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if not self.pg:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.device)
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return float(t.item())

    def gather(self, values) -> list:
        """Every rank's `values` (list of floats), as a list indexed by rank."""
        vals = [float(v) for v in values]
        if not self.pg:
            return [vals]
        t = self.torch.zeros((self.world, len(vals)), dtype=self.torch.float64,
                             device=self.device)
        t[self.rank] = self.torch.tensor(vals, dtype=self.torch.float64)
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return t.cpu().tolist()

    def close(self):
        if self.pg:
            self.td.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU: the reference on this host's cores
# ---------------------------------------------------------------------------
def _per_grid_seconds(cfg, fn) -> float:
    """Serial seconds per grid of `fn(packed_batch)` on 4 molecules (probe)."""
    from paper_2211_08506_b200 import synth

    probe = synth.packed_batch(cfg, range(4))
    t0 = time.perf_counter()
    fn(probe)
    return (time.perf_counter() - t0) / 4


def _stock_grid(cfg):
    from baseline import refbench

    vx = refbench._voxgrid()

    def run(pb):
        sets, spec = refbench._build(cfg, pb)
        for ps in sets:
            vx.generate_grid(ps, spec)
    return run


def cpu_sample_size(cfg, B, workers, seconds, per_grid) -> int:
    """Molecules for ~`seconds` of work on `workers` cores (the whole batch
    when it fits: same_config)."""
    return int(min(B, max(2 * workers, seconds * workers / max(per_grid, 1e-9))))


def cpu_reference(cfg, B, seconds: float, passes: int = 2):
    """The stock reference (baseline/_ref) as a process pool over
    generate_grid on (a prefix of) the same batch; None if not installed."""
    from baseline import refbench
    from paper_2211_08506_b200 import synth

    if not refbench.available():
        return None
    workers = refbench.host_cores()
    n = cpu_sample_size(cfg, B, workers, seconds / max(passes, 1), _per_grid_seconds(cfg, _stock_grid(cfg)))
    pb = synth.packed_batch(cfg, range(n))
    rate, dt, workers = refbench.time_pool(cfg, pb, passes=passes, warmup=1, workers=workers)
    same = n == B
    return {"value": rate, "unit": "grids/s", "cores": workers, "kind": "reference",
            "same_config": same,
            "sample": (f"{'the same' if same else 'the first'} {n} molecules of {cfg.name}"
                       f"{'' if same else f' (of {B})'}, {passes} timed passes after one untimed: "
                       f"process pool of {workers} over the stock voxgrid.generate_grid "
                       f"(baseline/_ref; grids dropped in the workers)"),
            **refbench.host_info()}


def cpu_port(cfg, B, seconds: float):
    """The oracle port (numpy restatement) on all host cores: process pool
    writing into shared memory."""
    from oracle import voxgrid_oracle as orc
    from paper_2211_08506_b200 import synth

    geom = orc.Geometry(cfg.shape, cfg.channels, cfg.box_origin, cfg.box_extents, cfg.sigma)
    workers = orc.host_cores()
    per = _per_grid_seconds(cfg, lambda pb: orc.batch(pb.offsets, pb.channels, pb.xyz, geom))
    n = cpu_sample_size(cfg, B, workers, seconds, per)
    pb = synth.packed_batch(cfg, range(n))
    pool = orc.Pool(geom, n, workers)
    try:
        # warm the workers and first-touch every page of the shared output
        pool.run(pb.offsets, pb.channels, pb.xyz)
        t0 = time.perf_counter()
        pool.run(pb.offsets, pb.channels, pb.xyz)
        dt = time.perf_counter() - t0
    finally:
        pool.close()
    return {"value": n / dt, "unit": "grids/s", "cores": workers, "kind": "port",
            "same_config": n == B,
            "sample": f"{n} molecules of {cfg.name} in {dt:.2f}s (numpy port of "
                      f"voxgrid.generate_grid, process pool of {workers} writing into shared memory)"}


def cpu_baseline(cfg, B, seconds: float):
    ref = cpu_reference(cfg, B, seconds)
    port = cpu_port(cfg, B, min(seconds, 4.0))
    if ref is None:
        return port
    ref["port"] = {k: port[k] for k in ("value", "cores", "sample")}
    return ref


def run_reference(args):
    """`--impl reference`: the unmodified reference on the host cores, rank 0
    only. Each step is one pass of the process pool over the stock
    generate_grid on the same batch as the GPU arm (a prefix of it when the
    whole batch would exceed ~2.5 s of CPU per step)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from baseline import refbench
    from paper_2211_08506_b200 import synth

    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.n_molecules
    H, W, D = cfg.shape
    if not refbench.available():
        return run_reference_port(args, cfg, B)
    workers = refbench.host_cores()
    n = cpu_sample_size(cfg, B, workers, 2.5, _per_grid_seconds(cfg, _stock_grid(cfg)))
    pb = synth.packed_batch(cfg, range(n))
    pool = refbench.RefPool(cfg, pb, workers)
    try:
        for _ in range(args.warmup):
            pool.run()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.run()
        dt = time.perf_counter() - t0
    finally:
        pool.close()
    rate = n * args.steps / dt
    # the reference's own parallel API on (a bounded prefix of) the same batch
    per1 = _per_grid_seconds(cfg, _stock_grid(cfg))
    n_gb = int(min(n, max(workers, 8.0 / max(per1, 1e-9))))
    gb_rate, gb_dt, _ = refbench.time_generate_batch(cfg, synth.packed_batch(cfg, range(n_gb)),
                                                     workers)
    same = n == B
    sample = (f"{'the same' if same else 'the first'} {n} molecules of {cfg.name} per step: "
              f"process pool of {workers} over the stock voxgrid.generate_grid (baseline/_ref)")
    line = {
        "impl": "reference", "metric": "grids_per_sec", "value": rate, "unit": "grids/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "voxels_per_sec": rate * cfg.channels * H * W * D,
        "config": {"workload": f"{cfg.name}: {n} molecules per step on the CPU",
                   "global_batch": B, "grid": [cfg.channels, H, W, D], "sigma": cfg.sigma,
                   "same_config": same},
        "cpu_baseline": {"value": rate, "unit": "grids/s", "cores": workers, "kind": "reference",
                         "sample": sample, **refbench.host_info()},
        "reference_generate_batch": {
            "value": gb_rate, "unit": "grids/s", "threads": workers,
            "sample": f"voxgrid.generate_batch(parallelism={workers}) over the first {n_gb} "
                      f"molecules in {gb_dt:.2f}s (ThreadPoolExecutor, GIL-bound)"},
        "e2e": {"value": rate, "unit": "grids/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference_port(args, cfg, B):
    """Reference arm without baseline/_ref: the oracle port on the host cores."""
    from oracle import voxgrid_oracle as orc
    from paper_2211_08506_b200 import synth

    geom = orc.Geometry(cfg.shape, cfg.channels, cfg.box_origin, cfg.box_extents, cfg.sigma)
    workers = orc.host_cores()
    per = _per_grid_seconds(cfg, lambda pb: orc.batch(pb.offsets, pb.channels, pb.xyz, geom))
    n = cpu_sample_size(cfg, B, workers, 2.5, per)
    pb = synth.packed_batch(cfg, range(n))
    pool = orc.Pool(geom, n, workers)
    try:
        for _ in range(args.warmup):
            pool.run(pb.offsets, pb.channels, pb.xyz)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.run(pb.offsets, pb.channels, pb.xyz)
        dt = time.perf_counter() - t0
    finally:
        pool.close()
    rate = n * args.steps / dt
    H, W, D = cfg.shape
    sample = (f"{n} molecules of {cfg.name} per step (numpy port of voxgrid.generate_grid, "
              f"process pool of {workers} writing into shared memory; baseline/_ref missing)")
    line = {
        "impl": "reference", "metric": "grids_per_sec", "value": rate, "unit": "grids/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "voxels_per_sec": rate * cfg.channels * H * W * D,
        "config": {"workload": f"{cfg.name}: CPU sample of {n} molecules per step",
                   "global_batch": B, "grid": [cfg.channels, H, W, D], "sigma": cfg.sigma,
                   "same_config": n == B},
        "cpu_baseline": {"value": rate, "unit": "grids/s", "cores": workers, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "grids/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_b200(args):
    import torch

    world, rank, local = dist_env()
    n_dev = torch.cuda.device_count()
    if n_dev < 1:
        raise SystemExit("bench.py: no CUDA device (use --dry-run for the CPU plumbing test)")
    shared = world > n_dev               # ranks share GPUs (plumbing runs on a 1-GPU box)
    local = local % n_dev
    torch.cuda.set_device(local)
    backend = args.dist_backend
    if backend == "auto":
        backend = "gloo" if shared else "nccl"   # NCCL refuses two ranks on one device
    dist = Dist(world, rank, local, backend=backend)
    import paper_2211_08506_b200 as vg
    from paper_2211_08506_b200 import _native, synth

    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.n_molecules
    indices = plan_indices(cfg, B, rank, world, args.scaling)
    t0 = time.perf_counter()
    pb = synth.packed_batch(cfg, indices)
    log(f"[bench rank{rank}] synthesized {pb.n_molecules} molecules / {len(pb.channels)} atoms "
        f"in {time.perf_counter() - t0:.1f}s")
    Bl = pb.n_molecules
    H, W, D = cfg.shape
    spec = vg.GridSpec(cfg.shape, cfg.channels, vg.BoundingBox(cfg.box_origin, cfg.box_extents),
                       cfg.sigma)
    dev = torch.device("cuda", local)
    eng = vg.GridEngine(dev)
    lib = _native.lib()
    stream = torch.cuda.current_stream(dev)

    # device-resident inputs for the `value` leg
    off_d = torch.from_numpy(pb.offsets).to(dev)
    ch_d = torch.from_numpy(pb.channels).to(dev)
    xyz_d = torch.from_numpy(pb.xyz).to(dev)
    out = torch.empty((Bl, cfg.channels, H, W, D), dtype=torch.float32, device=dev)
    stats = torch.empty((Bl, 2), dtype=torch.int64, device=dev)
    desc = eng.describe(off_d, ch_d, xyz_d, spec)
    layout = _native.VgWsLayout()
    _native.check(lib.vg_workspace_layout(desc, layout), "layout")
    ws = torch.empty(layout.total, dtype=torch.uint8, device=dev)
    sptr = stream.cuda_stream

    # small batches run one kernel (K13: tables in shared memory + gather);
    # the others K1 (tables) then K3 (slabs), timed separately
    fused = lib.vg_fused_small(desc, out.data_ptr()) == 1

    def step():
        if fused:
            _native.check(lib.vg_generate_f32(desc, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                              stats.data_ptr(), sptr), "generate")
            return
        _native.check(lib.vg_axis_tables_f32(desc, ws.data_ptr(), ws.numel(), sptr), "tables")
        _native.check(lib.vg_slabs_f32(desc, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       stats.data_ptr(), sptr), "slabs")

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    K = args.steps
    # Steps whose output fits the L2 (cfg0: 42 MB of a 126 MB L2) would time
    # L2-resident writes: flush the L2 before every step (a 4 x L2 store
    # stream, outside the step's events) and take the flushed serial rate.
    l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20))
    flush = Bl * cfg.grid_bytes < 2 * l2_bytes
    scratch = torch.empty(4 * l2_bytes // 4, dtype=torch.float32, device=dev) if flush else None

    def flush_l2(st):
        if flush:
            _native.check(lib.vg_fill_f32(scratch.data_ptr(), scratch.numel(), 0.0, st), "flush")

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    sampler = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for k in range(K):
            flush_l2(sptr)
            ev[k][0].record(stream)
            if fused:   # one kernel: its time is the step's (k1 = 0)
                ev[k][1].record(stream)
                _native.check(lib.vg_generate_f32(desc, out.data_ptr(), ws.data_ptr(),
                                                  ws.numel(), stats.data_ptr(), sptr), "generate")
            else:
                _native.check(lib.vg_axis_tables_f32(desc, ws.data_ptr(), ws.numel(), sptr),
                              "tables")
                ev[k][1].record(stream)
                _native.check(lib.vg_slabs_f32(desc, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                               stats.data_ptr(), sptr), "slabs")
            ev[k][2].record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    k1_ms = [e[0].elapsed_time(e[1]) for e in ev]
    k3_ms = [e[1].elapsed_time(e[2]) for e in ev]
    pairs = int(stats[:, 0].sum().item())    # P = sum of voxel_writes
    total_ms = (sum(a + b for a, b in zip(k1_ms, k3_ms)) if flush
                else ev[0][0].elapsed_time(ev[-1][2]))
    step_api = "vg_axis_tables_f32 + vg_slabs_f32 (K1 and K3 timed apart)"
    if flush and not fused:
        # L2-flushed steps are timed one by one: time them through the
        # product's serial entry point, vg_generate_f32 (K3 launched as K1's
        # programmatic dependent); the K1 / K3 split above stays the roofline's
        gv = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        with sampler:
            for k in range(K):
                flush_l2(sptr)
                gv[k][0].record(stream)
                _native.check(lib.vg_generate_f32(desc, out.data_ptr(), ws.data_ptr(),
                                                  ws.numel(), stats.data_ptr(), sptr), "generate")
                gv[k][1].record(stream)
            torch.cuda.synchronize()
        total_ms = sum(a.elapsed_time(b) for a, b in gv)
        step_api = "vg_generate_f32 (K1, then K3 as its programmatic dependent)"
    t_max_serial = dist.max(total_ms)
    grids_total = dist.sum(float(Bl)) * K
    value_serial = grids_total / (t_max_serial / 1e3)

    # `value`: the same K steps through the pipelined path (K1 of step k+1 on
    # its own stream, concurrent with K3 of step k), inputs resident in HBM
    from paper_2211_08506_b200.loader import GridPipeline, pinned_csr

    pipe = GridPipeline(spec, dev)
    for _ in range(max(args.warmup, 3)):
        pipe.submit(off_d, ch_d, xyz_d)
    pipe.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    pa, pb_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = pipe.launches
    with sampler:
        pa.record(pipe.compute_stream)
        pipe.begin(pa)
        for _ in range(K):
            pipe.submit(off_d, ch_d, xyz_d)
        pb_.record(pipe.join())   # after the K3s of every slot's compute stream
        torch.cuda.synchronize()
    pipe_ms = pa.elapsed_time(pb_)
    t_max = dist.max(pipe_ms)
    value = grids_total / (t_max / 1e3)
    if flush:   # the overlapped loop would run L2-warm: report the flushed serial rate
        value_l2_warm, value, t_max = value, value_serial, t_max_serial
    launches = pipe.launches - launches0   # kernels the library reports (K1, K2 if binned, K3)

    # roofline of K3 (dominant kernel): algorithmic bytes = the output grids
    alg_bytes = Bl * cfg.grid_bytes
    k3_avg = statistics.mean(k3_ms)
    achieved = alg_bytes / (k3_avg / 1e3) / 1e9
    peak, peak_src = peaks()

    # pure-write fill of the same bytes: what HBM sustains for stores alone
    for _ in range(3):
        _native.check(lib.vg_fill_f32(out.data_ptr(), out.numel(), 0.0, sptr), "fill")
    fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fa.record(stream)
    for _ in range(5):
        _native.check(lib.vg_fill_f32(out.data_ptr(), out.numel(), 0.0, sptr), "fill")
    fb.record(stream)
    torch.cuda.synchronize()
    fill_gbs = alg_bytes * 5 / (fa.elapsed_time(fb) / 1e3) / 1e9

    # e2e through the public pipelined API: pinned host CSR -> H2D (copy
    # stream) -> K1 -> K3 -> D2H of the per-grid stats, every step
    off_h, ch_h, xyz_h = pinned_csr(pb.offsets, pb.channels, pb.xyz)
    st_h = torch.empty((Bl, 2), dtype=torch.int64).pin_memory()
    h2d = off_h.numel() * 8 + ch_h.numel() * 4 + xyz_h.numel() * 8
    d2h = st_h.numel() * 8
    epipe = pipe  # reuse its double buffers (large configs: 2 x 43 GB at cfg2)

    def e2e_step():
        # H2D of the CSR inputs, K1, K2/K3 and the D2H of the stats: one native call
        epipe.submit(off_h, ch_h, xyz_h, stats_out=st_h)

    for _ in range(max(args.warmup, 3)):
        e2e_step()
    epipe.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if flush:
        # L2 flushed before every step: steps run one at a time, each timed
        # from its submit to its stats on the host (flushes not timed)
        wall, e2e_event_ms = 0.0, 0.0
        for _ in range(K):
            flush_l2(epipe.compute_stream.cuda_stream)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            ea.record(epipe.compute_stream)
            epipe.begin(ea)
            e2e_step()
            epipe.compute_stream.wait_stream(epipe.readback_stream)   # stats on the host
            eb.record(epipe.compute_stream)
            eb.synchronize()
            wall += time.perf_counter() - w0
            e2e_event_ms += ea.elapsed_time(eb)
    else:
        w0 = time.perf_counter()
        ea.record(epipe.compute_stream)
        epipe.begin(ea)
        for _ in range(K):
            e2e_step()
        epipe.compute_stream.wait_stream(epipe.readback_stream)   # last stats on the host
        eb.record(epipe.compute_stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        e2e_event_ms = ea.elapsed_time(eb)
    e2e_ms = max(e2e_event_ms, wall * 1e3)
    e2e_value = grids_total / (dist.max(e2e_ms) / 1e3)
    dist.barrier()

    # The reference-facing API on the same batch: GaussianVoxelizer.transform
    # over (m, 4) host arrays (validation, packing, H2D and K1 + K3 per call),
    # with a D2H of one voxel per grid as the read-back; steps one after the
    # other (rank 0, single GPU only: informational)
    transform = None
    if world == 1 and not flush:
        X = [np.column_stack([pb.channels[a:b].astype(np.float64), pb.xyz.reshape(-1, 3)[a:b]])
             for a, b in zip(pb.offsets[:-1], pb.offsets[1:])]
        est = vg.GaussianVoxelizer(grid_size=cfg.shape, sigma=cfg.sigma, n_channels=cfg.channels,
                                   box=(cfg.box_origin, cfg.box_extents)).fit(X)
        for _ in range(2):
            est.transform(X)[:, 0, 0, 0, 0].cpu()
        torch.cuda.synchronize()
        # (a) blocking: every call's read-back waits for its grids
        t0 = time.perf_counter()
        for _ in range(K):
            est.transform(X)[:, 0, 0, 0, 0].cpu()
        dt_sync = (time.perf_counter() - t0) / K
        # (b) a loader's use: every call's read-back is queued (pinned host
        # buffer, non-blocking) and the host validates and packs the next
        # call while the device works; all read-backs complete before the clock
        # stops
        heads = torch.empty((K, Bl), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(K):
            heads[k].copy_(est.transform(X)[:, 0, 0, 0, 0], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / K
        transform = {"value": Bl / dt, "unit": "grids/s", "ms_per_step_wall": dt * 1e3,
                     "value_blocking": Bl / dt_sync, "ms_per_step_wall_blocking": dt_sync * 1e3,
                     "h2d_bytes_per_step": int(len(pb.channels) * 32),
                     "d2h_bytes_per_step": Bl * 4,
                     "api": "paper_2211_08506_b200.GaussianVoxelizer.transform(list of (m,4) "
                            "numpy arrays) + D2H of one voxel per grid: queued into pinned "
                            "memory per call (value) or blocking per call (value_blocking)"}

    # per rank: molecules, pipelined ms/step, K3 ms, K3 GB/s (max-over-ranks
    # timing is what `value` uses; this shows the balance)
    per_rank = dist.gather([Bl, pipe_ms / K, k3_avg, achieved, len(pb.channels)])
    sm_mhz = sampler.summary().get("sm_mhz")
    compute = compute_leg(cfg, Bl, len(pb.channels), pairs, alg_bytes, peak, sm_mhz, dev)
    line = None
    if rank == 0:
        n_atoms = len(pb.channels)
        line = {
            "metric": "grids_per_sec",
            "value": value,
            "unit": "grids/s",
            "n_gpus": world,
            "ranks_per_gpu": (world + n_dev - 1) // n_dev if shared else 1,
            "steps": K,
            "warmup": max(args.warmup, 3),
            "ms_per_step": t_max / K,
            "value_serial": value_serial,
            "ms_per_step_serial": t_max_serial / K,
            "serial_step_api": step_api,
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": "f32",
            "grids_per_sec_per_gpu": value / world,
            "data": "synthetic (seeded BASELINE config distribution; no dataset)",
            "voxels_per_sec": value * cfg.channels * H * W * D,
            "config": {
                "workload": f"{cfg.name}: {int(grids_total / K)} molecules -> fp32 "
                            f"[{int(grids_total / K)},{cfg.channels},{H},{W},{D}], sigma "
                            f"{cfg.sigma}, box {cfg.box_extents[0]} A"
                            + (f", {args.scaling} scaling over {world} ranks" if world > 1 else ""),
                "global_batch": int(grids_total / K),
                "grid": [cfg.channels, H, W, D],
                "atoms_rank0": n_atoms,
                "parallelism": f"molecule-sharded x{world} (cost-balanced contiguous ranges), "
                               f"no collective; timing plumbing over {backend}",
                "pipeline": f"GridPipeline depth {len(pipe.slots)}, {len(pipe.compute_streams)} "
                            "compute streams (one per slot: consecutive K3s overlap their tails); "
                            "value_serial runs K1 then K3 on one stream",
                "l2": (f"flushed: each step writes {alg_bytes / 1e6:.0f} MB, which fits the "
                       f"{l2_bytes >> 20} MB L2, so a {4 * l2_bytes >> 20} MB store stream runs "
                       "before every timed step (not timed); value and e2e are then per-step "
                       "serial rates" if flush else
                       f"no flush needed: each step writes {alg_bytes / 1e9:.2f} GB, "
                       f"> {l2_bytes >> 20} MB L2"),
            },
            "per_rank": [{"rank": r, "molecules": int(v[0]), "atoms": int(v[4]),
                          "ms_per_step": v[1], "grids_per_sec": v[0] / (v[1] / 1e3) if v[1] else None,
                          "k3_ms": v[2], "k3_gbs": v[3], "k3_frac": v[3] / peak}
                         for r, v in enumerate(per_rank)],
            "roofline": {
                "bound": compute["bound"],
                "kernel": ("vg_small_kernel (K13: axis tables in shared memory + gather, "
                           "one launch)" if fused else "vg_slab_kernel (K3)"),
                # per GPU: rank 0's K3 (per_rank lists every GPU's)
                "achieved": achieved,
                "peak": peak,
                "peak_source": peak_src,
                "unit": "GB/s",
                "frac": achieved / peak,
                "frac_min_over_gpus": min(v[3] for v in per_rank) / peak,
                "compute": compute,
                "traffic": traffic_from_profiles(args.config),
                "alg_bytes_per_launch": alg_bytes,
                "k3_ms": k3_avg,
                "k1_ms": statistics.mean(k1_ms),
                "k3_share_of_step": k3_avg / (total_ms / K),
                "k3_share_of_pipelined_step": k3_avg / (pipe_ms / K),
                "write_fill_gbs": fill_gbs,
                # the measured peak is a copy (read + write) rate; a pure
                # 128-bit store stream runs faster, so frac can exceed 1:
                # this is K3 against the write ceiling measured in this run
                "frac_vs_write_fill": achieved / fill_gbs,
            },
            "e2e": {"value": e2e_value, "unit": "grids/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "ms_per_step_event": e2e_event_ms / K, "ms_per_step_wall": wall * 1e3 / K,
                    "api": "paper_2211_08506_b200.loader.GridPipeline.submit(pinned host CSR)"},
            "gpu_launches": launches,
            "clocks": sampler.summary(),
        }
        if transform is not None:
            line["e2e_transform"] = transform
        if flush:   # for reference only: the overlapped loop with the output in L2
            line["value_pipelined_l2_warm"] = value_l2_warm
    dist.close()
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, B, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    return 0


def compute_leg(cfg, n_mol, n_atoms, pairs, alg_bytes, hbm_gbs, sm_mhz, dev):
    """The other two legs of the north_star roofline: the FP32
    and SFU time of the Gaussian evaluation, from the algorithmic counts
    P = sum of voxel_writes (3 flops per pair: two multiplies and the add) and
    E = erf_evals = atoms x ((W+1)+(H+1)+(D+1)) (~20 flops and 3 SFU ops
    (ex2, sqrt, rcp) each), against 148 SMs x 128 FP32 lanes x 2 and 16 SFU
    lanes per SM at the sampled SM clock. The roofline time is the largest."""
    import torch

    H, W, D = cfg.shape
    evals = n_atoms * ((W + 1) + (H + 1) + (D + 1))
    flops = 3 * pairs + 20 * evals
    sfu = 3 * evals
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    ghz = (sm_mhz or 1965.0) / 1e3
    fp32_peak = sms * 128 * 2 * ghz * 1e9
    sfu_peak = sms * 16 * ghz * 1e9
    t_hbm = alg_bytes / (hbm_gbs * 1e9)
    t_fp32 = flops / fp32_peak
    t_sfu = sfu / sfu_peak
    bound = max((t_hbm, "hbm"), (t_fp32, "fp32"), (t_sfu, "sfu"))[1]
    return {"bound": bound, "pairs": pairs, "erf_evals": evals, "flops": flops, "sfu_ops": sfu,
            "t_hbm_ms": t_hbm * 1e3, "t_fp32_ms": t_fp32 * 1e3, "t_sfu_ms": t_sfu * 1e3,
            "fp32_tflops_peak": fp32_peak / 1e12, "sfu_tops_peak": sfu_peak / 1e12,
            "sm_count": sms, "sm_ghz": ghz}


def traffic_from_profiles(config: int):
    """dram bytes per K3 launch from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(f"cfg{config}")
    except Exception:  # noqa: BLE001
        return None


def run_dry(args):
    """--dry-run: the multi-rank plumbing without kernels (CPU, gloo): shard
    plan, per-rank synthesis, barrier, max/sum/gather over ranks."""
    world, rank, local = dist_env()
    dist = Dist(world, rank, local, backend="gloo")
    from paper_2211_08506_b200 import synth

    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.n_molecules
    indices = plan_indices(cfg, B, rank, world, args.scaling)
    pb = synth.packed_batch(cfg, indices)
    dist.barrier()
    t0 = time.perf_counter()
    checksum = float(pb.xyz.sum())
    dt_ms = (time.perf_counter() - t0) * 1e3
    per_rank = dist.gather([pb.n_molecules, indices.start, indices.stop, len(pb.channels), dt_ms])
    total = dist.sum(float(pb.n_molecules))
    t_max = dist.max(dt_ms)
    dist.barrier()
    if rank == 0:
        print(json.dumps({
            "metric": "grids_per_sec", "dry_run": True, "value": None, "unit": "grids/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "scaling": args.scaling, "global_batch": int(total), "t_max_ms": t_max,
            "config": {"workload": cfg.name, "global_batch": int(total)},
            "per_rank": [{"rank": r, "molecules": int(v[0]), "start": int(v[1]),
                          "stop": int(v[2]), "atoms": int(v[3])} for r, v in enumerate(per_rank)],
            "checksum_rank0": checksum}), flush=True)
    dist.close()
    return 0


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        return run_reference(args)          # rank 0 alone, host cores
    if env_world is None:
        if args.gpus > 1:
            return spawn_ranks(args.gpus)   # one process per GPU
    elif int(env_world) != args.gpus:
        print(f"bench.py: WORLD_SIZE={env_world} but --gpus {args.gpus}; launch one rank per "
              "GPU with matching counts", file=sys.stderr)
        return 2
    if args.dry_run:
        return run_dry(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
