"""The C-ABI library on a CPU-only host: it loads, exports every symbol the
public header declares, and its host build of the device numerics (shared
source csrc/vg_math.cuh) reproduces numpy's float32 exp and the reference
erf bit for bit. No compute call touches a GPU here."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from _golden import erf_cases
from oracle import voxgrid_oracle as orc
from paper_2211_08506_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "voxgrid_b200.h"


@pytest.fixture(scope="module")
def lib():
    _native.build_native()
    return _native.lib()


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(vg_\w+)\s*\(", text, re.M)))


def test_header_declares_expected_api():
    names = declared_functions()
    for must in ("vg_generate_f32", "vg_workspace_layout", "vg_axis_tables_f32", "vg_erf_f32",
                 "vg_exp_f32_host", "vg_erf_f32_host", "vg_last_error", "vg_abi_version",
                 "vg_fill_f32"):
        assert must in names
    assert set(names) == set(_native.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.vg_abi_version() == _native.ABI_VERSION


def _host(fn, x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    assert fn(x.ctypes.data, out.ctypes.data, x.size) == 0
    return out


def test_host_exp_matches_numpy_sample_of_all_floats(lib):
    bits = np.arange(0, 2**32, 61, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    with np.errstate(all="ignore"):
        ref = np.exp(x)
    got = _host(lib.vg_exp_f32_host, x)
    same = (got.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(got) & np.isnan(ref))
    assert same.all(), f"{(~same).sum()} mismatches, first at {x[~same][:4]}"


def test_host_exp_matches_numpy_on_erf_domain(lib):
    # y = -t*t in (-17, 0] is where exp's bits reach the Bürmann erf
    lo = int(np.float32(-17.0).view(np.uint32))
    bits = np.arange(0x80000000, lo + 1, 13, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    assert np.array_equal(_host(lib.vg_exp_f32_host, x).view(np.uint32),
                          np.exp(x).view(np.uint32))


def test_host_erf_matches_golden_reference_values(lib):
    t, e = erf_cases()
    assert np.array_equal(_host(lib.vg_erf_f32_host, t).view(np.uint32), e.view(np.uint32))


def test_host_erf_matches_oracle_dense_range(lib):
    hi = int(np.float32(6.0).view(np.uint32))
    t = np.arange(0, hi, 37, dtype=np.uint32).view(np.float32)
    t = np.concatenate([t, -t])
    with np.errstate(all="ignore"):
        ref = orc.erf_f32(t)
    assert np.array_equal(_host(lib.vg_erf_f32_host, t).view(np.uint32), ref.view(np.uint32))


def test_erf_saturates_exactly(lib):
    # reference test_kernels.py:54 — erf(5.0f) == 1.0f exactly; odd symmetry exact
    t = np.array([5.0, -5.0, 0.0, -0.0, 9.0], dtype=np.float32)
    got = _host(lib.vg_erf_f32_host, t)
    assert got[0] == 1.0 and got[1] == -1.0 and got[2] == 0.0 and got[4] == 1.0


def test_invalid_descriptor_reports_error_without_gpu(lib):
    d = _native.VgBatchDesc()
    d.n_molecules, d.n_atoms = 1, 0
    d.H = d.W = d.D = 0
    d.C = 1
    d.scale = 1.0
    layout = _native.VgWsLayout()
    rc = lib.vg_workspace_layout(ctypes.byref(d), ctypes.byref(layout))
    assert rc == -1
    assert b"shape" in lib.vg_last_error()
    d.H = d.W = d.D = 8
    d.delta[:] = (0.5, 0.5, 0.5)
    d.offsets = 8  # any non-NULL pointer; layout never dereferences it
    assert lib.vg_workspace_layout(ctypes.byref(d), ctypes.byref(layout)) == 0
    assert layout.total >= 256 and layout.row_x == 8


def test_launch_planning_every_forced_cta_width(lib, monkeypatch):
    """The K3 launch plan (run by vg_workspace_layout on the host, no GPU)
    for every forced thread multiple VG_PLAN_Q, including ones its rules
    reject (they fall back to the free choice instead of leaving the plan
    empty), and every shape class of the BASELINE configs."""
    d = _native.VgBatchDesc()
    d.C = 5
    d.scale = 1.0
    d.offsets = 8   # any non-NULL pointer; planning never dereferences it
    layout = _native.VgWsLayout()
    for shape in ((32, 32, 32), (64, 64, 64), (48, 48, 48), (128, 128, 128), (5, 7, 9)):
        d.H, d.W, d.D = shape
        d.delta[:] = (0.3, 0.3, 0.3)
        for atoms in (19, 2000):
            d.n_molecules, d.n_atoms = 4, 4 * atoms
            d.xyz = d.channel = 8
            for q in ("", "1", "2", "3", "4", "5", "8", "16"):
                monkeypatch.setenv("VG_PLAN_Q", q)
                assert lib.vg_workspace_layout(ctypes.byref(d), ctypes.byref(layout)) == 0
                assert layout.total >= 256


def test_erf_saturation_threshold(lib):
    """K1 skips the series where E(t) is exactly +-1: E(t) == 1.0f for every
    float32 t >= t_sat (checked on every float in [t_sat, t_sat*4) and a
    sample up to +inf), and E(prev(t_sat)) < 1."""
    tsat = np.float32(float.fromhex("0x1.01a2a2p+2"))
    below = np.nextafter(tsat, np.float32(0), dtype=np.float32)
    lo = int(tsat.view(np.uint32))
    dense = np.arange(lo, lo + (2 << 23), dtype=np.uint32).view(np.float32)
    sparse = np.arange(lo, 0x7F800001, 9973, dtype=np.uint64).astype(np.uint32).view(np.float32)
    for t in (dense, sparse):
        assert np.all(_host(lib.vg_erf_f32_host, t) == 1.0)
        assert np.all(_host(lib.vg_erf_f32_host, -t) == -1.0)
    assert _host(lib.vg_erf_f32_host, np.array([below], np.float32))[0] < 1.0


def test_saturated_erf_equals_full_erf(lib):
    """K1's vg_erf_sat_f32 (range checks of exp dropped inside |t| < t_sat)
    is bit-identical to vg_erf_f32 on a strided sample of every float in
    (-t_sat, t_sat), the neighbourhood of +-t_sat, zeros, infinities and NaN.
    (The full 2^31-float sweep was run once when it was introduced.)"""
    tsat = np.float32(float.fromhex("0x1.01a2a2p+2"))
    hi = int(tsat.view(np.uint32))
    pos = np.arange(0, hi + 4096, 61, dtype=np.uint32).view(np.float32)
    near = np.arange(hi - 4096, hi + 4096, dtype=np.uint32).view(np.float32)
    special = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, 3.0, 4.0255513], np.float32)
    for t in (pos, -pos, near, -near, special):
        a = _host(lib.vg_erf_sat_f32_host, t)
        b = _host(lib.vg_erf_f32_host, t)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    nan = _host(lib.vg_erf_sat_f32_host, np.array([np.nan], np.float32))
    assert np.isnan(nan[0])


def test_submit_validates_before_touching_the_gpu(lib):
    """vg_submit_f32 rejects NULL args and reports the workspace it needs
    before any CUDA call (so this runs without a GPU)."""
    import ctypes

    d = _native.VgBatchDesc()
    d.n_molecules, d.n_atoms = 2, 5
    d.offsets, d.xyz, d.channel = 16, 16, 16   # never dereferenced on these paths
    d.delta[:] = (0.5, 0.5, 0.5)
    d.scale = 1.0
    d.H = d.W = d.D = 8
    d.C = 3
    d.threshold = float("nan")
    assert lib.vg_submit_f32(d, None, 16, None, 0, None) == -1
    need = ctypes.c_size_t(0)
    args = _native.VgSubmitArgs()
    args.ws_needed = ctypes.pointer(need)
    assert lib.vg_submit_f32(d, args, 16, None, 0, None) == _native.VG_ERR_WORKSPACE
    layout = _native.VgWsLayout()
    assert lib.vg_workspace_layout(d, layout) == 0
    assert need.value == layout.total > 0


def test_descent_entry_points_validate_arguments(lib):
    """The device-descent calls reject NULL buffers and empty sizes before any
    launch (no GPU needed)."""
    assert lib.vg_descent_candidates_f64(None, 8, 8, 8, 8, 3, 11, 10, 1e-12, None) == -1
    assert lib.vg_descent_candidates_f64(8, 8, 8, 8, 8, 0, 11, 10, 1e-12, None) == -1
    assert lib.vg_descent_select_f64(8, 8, 8, 8, 3, 11, 100, 0, 8, 8, 8, None) == -1
    assert lib.vg_descent_select_f64(8, None, 8, 8, 3, 11, 100, 10, 8, 8, 8, None) == -1
    assert _native.VgDescentState.__dict__ and ctypes_sizeof_state() == 48


def ctypes_sizeof_state():
    import ctypes

    return ctypes.sizeof(_native.VgDescentState)


def _sass_by_function():
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "-sass", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        if "Function : " in line:
            cur = line.split("Function : ", 1)[1].strip()
            funcs[cur] = []
        elif cur is not None:
            funcs[cur].append(line)
    return funcs


def test_accumulation_is_never_contracted_to_fma(lib):
    """Bit parity needs acc + fl(fl(gy*gx)*gz) with two roundings: no kernel
    that accumulates voxels may contain FFMA / FFMA2. (ptxas 12.9 contracts
    mul.rn.f32x2 + add.rn.f32x2 into FFMA2 despite the rounding modifiers and
    --fmad=false; the packed forms are not used, profiles/r2_fmul2_ab.txt.)
    K1 / erf keep the FMAs of numpy's exp algorithm on purpose (vg_math.cuh)."""
    funcs = _sass_by_function()
    acc = {n: body for n, body in funcs.items()
           if any(k in n for k in ("vg_slab_kernel", "vg_slab_generic_kernel",
                                   "vg_slab_ws_kernel"))}
    assert len(acc) >= 20, sorted(funcs)[:5]
    for name, body in acc.items():
        text = "\n".join(body)
        assert "FFMA" not in text, name
    for name, body in funcs.items():
        if "vg_small_kernel" in name:
            assert "FFMA2" not in "\n".join(body), name


def test_slab_kernel_stages_with_bulk_copies_and_streaming_stores(lib):
    """The shipped K3 instances carry what DESIGN.md §5 describes: bulk-copy
    staging (UBLKCP) awaited on an mbarrier (SYNCS ... TRYWAIT), the cp.async
    path for unaligned rounds (LDGSTS) and 128-bit evict-first stores."""
    funcs = _sass_by_function()
    k3 = {n: "\n".join(b) for n, b in funcs.items() if "vg_slab_kernelILi1ELi8ELi2E" in n}
    assert len(k3) == 1, sorted(funcs)[:5]
    text = next(iter(k3.values()))
    for needle in ("UBLKCP", "SYNCS.ARRIVE", "TRYWAIT", "LDGSTS", "STG.E.EF.128"):
        assert needle in text, needle
