"""ctypes binding of the C-ABI in include/voxgrid_b200.h (libvoxgrid_b200.so).

The shared library is built in-tree by ``build_native()`` (nvcc, sm_100a)
and loaded once per process. There is no fallback: if the library is
missing every GPU entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
INCLUDE = REPO_DIR / "include"
LIB_PATH = Path(os.environ.get("VG_LIB", PKG_DIR / "libvoxgrid_b200.so"))  # VG_LIB: A/B builds

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-fmad=false",           # never contract mul+add: bit parity with numpy
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-shared",
]

VG_OK = 0
VG_ERR_INVALID = -1
VG_ERR_WORKSPACE = -3


class NativeUnavailable(ImportError):
    """The sm_100a extension is not built or cannot be loaded."""


class VgBatchDesc(ctypes.Structure):
    _fields_ = [
        ("n_molecules", ctypes.c_int64),
        ("n_atoms", ctypes.c_int64),
        ("offsets", ctypes.c_void_p),
        ("xyz", ctypes.c_void_p),
        ("channel", ctypes.c_void_p),
        ("mol_origin", ctypes.c_void_p),
        ("mol_delta", ctypes.c_void_p),
        ("origin", ctypes.c_double * 3),
        ("delta", ctypes.c_double * 3),
        ("scale", ctypes.c_double),
        ("threshold", ctypes.c_float),
        ("periodic", ctypes.c_int32),
        ("H", ctypes.c_int32),
        ("W", ctypes.c_int32),
        ("D", ctypes.c_int32),
        ("C", ctypes.c_int32),
    ]


class VgWsLayout(ctypes.Structure):
    _fields_ = [
        ("tx", ctypes.c_size_t),
        ("ty", ctypes.c_size_t),
        ("tz", ctypes.c_size_t),
        ("supp", ctypes.c_size_t),
        ("total", ctypes.c_size_t),
        ("row_x", ctypes.c_int32),
        ("row_y", ctypes.c_int32),
        ("row_z", ctypes.c_int32),
        ("bins", ctypes.c_size_t),
        ("bin_off", ctypes.c_size_t),
        ("bin_jc", ctypes.c_int32),
        ("bin_chunks", ctypes.c_int32),
    ]


class VgSubmitArgs(ctypes.Structure):
    _fields_ = [
        ("h_offsets", ctypes.c_void_p),
        ("h_channel", ctypes.c_void_p),
        ("h_xyz", ctypes.c_void_p),
        ("h_stats", ctypes.c_void_p),
        ("copy_stream", ctypes.c_void_p),
        ("tables_stream", ctypes.c_void_p),
        ("compute_stream", ctypes.c_void_p),
        ("ev_wait", ctypes.c_void_p),
        ("ev_copied", ctypes.c_void_p),
        ("ev_tabled", ctypes.c_void_p),
        ("ev_done", ctypes.c_void_p),
        ("ws_needed", ctypes.POINTER(ctypes.c_size_t)),
        ("kernels", ctypes.POINTER(ctypes.c_int32)),
        ("readback_stream", ctypes.c_void_p),
        ("ev_read", ctypes.c_void_p),
    ]


class VgDescentState(ctypes.Structure):
    _fields_ = [
        ("current", ctypes.c_double),
        ("best", ctypes.c_double),
        ("iterations", ctypes.c_int64),
        ("forced", ctypes.c_int64),
        ("done", ctypes.c_int32),
        ("diverged", ctypes.c_int32),
        ("sel", ctypes.c_int32),
        ("moved", ctypes.c_int32),
    ]


# name -> (restype, argtypes); every symbol include/voxgrid_b200.h declares
SIGNATURES = {
    "vg_workspace_layout": (ctypes.c_int, [ctypes.POINTER(VgBatchDesc), ctypes.POINTER(VgWsLayout)]),
    "vg_generate_f32": (ctypes.c_int, [ctypes.POINTER(VgBatchDesc), ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                       ctypes.c_void_p]),
    "vg_slabs_f32": (ctypes.c_int, [ctypes.POINTER(VgBatchDesc), ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                    ctypes.c_void_p]),
    "vg_submit_f32": (ctypes.c_int, [ctypes.POINTER(VgBatchDesc), ctypes.POINTER(VgSubmitArgs),
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_void_p]),
    "vg_axis_tables_f32": (ctypes.c_int, [ctypes.POINTER(VgBatchDesc), ctypes.c_void_p,
                                          ctypes.c_size_t, ctypes.c_void_p]),
    "vg_fused_small": (ctypes.c_int, [ctypes.POINTER(VgBatchDesc), ctypes.c_void_p]),
    "vg_erf_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.c_void_p]),
    "vg_fill_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_float,
                                   ctypes.c_void_p]),
    "vg_mse_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32]),
    "vg_mse_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                  ctypes.c_void_p]),
    "vg_loss_gradient_f64": (ctypes.c_int, [ctypes.POINTER(VgBatchDesc), ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "vg_descent_candidates_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                                 ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                                 ctypes.c_void_p]),
    "vg_descent_select_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "vg_mse_grouped_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "vg_descent_candidates_batch_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                                       ctypes.c_int32, ctypes.c_void_p,
                                                       ctypes.c_void_p, ctypes.c_void_p,
                                                       ctypes.c_void_p, ctypes.c_int32,
                                                       ctypes.c_int64, ctypes.c_double,
                                                       ctypes.c_void_p]),
    "vg_descent_select_batch_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                   ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                   ctypes.c_void_p]),
    "vg_exp_f32_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "vg_erf_f32_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "vg_erf_sat_f32_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "vg_last_error": (ctypes.c_char_p, []),
    "vg_abi_version": (ctypes.c_int, []),
}

ABI_VERSION = 5
_lib = None


def build_native(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/*.cu into the in-tree shared library (sm_100a)."""
    sources = sorted(CSRC.glob("*.cu"))
    deps = sources + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    if not force and LIB_PATH.exists():
        newest = max(p.stat().st_mtime for p in deps)
        if LIB_PATH.stat().st_mtime >= newest:
            return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *NVCC_FLAGS, f"-I{INCLUDE}", "-o", str(tmp), *map(str, sources)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr}")
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def _pack_path() -> Path:
    import sysconfig

    return PKG_DIR / ("_vgpack" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pack(force: bool = False) -> Path:
    """Compile csrc/vg_pack.cpp (CPython extension ``_vgpack``: the host
    packer of the drop-in APIs) in-tree with g++."""
    import sysconfig

    src = CSRC / "vg_pack.cpp"
    out = _pack_path()
    if not force and out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    tmp = out.with_suffix(".so.tmp")
    import numpy

    cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-shared", "-fPIC",
           "-fvisibility=hidden", f"-I{sysconfig.get_paths()['include']}",
           f"-I{numpy.get_include()}", "-o", str(tmp), str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr}")
    os.replace(tmp, out)
    return out


_pack = None


def pack():
    """The ``_vgpack`` host packer module (built on first use if missing)."""
    global _pack
    if _pack is None:
        import importlib.util

        path = build_pack()
        spec = importlib.util.spec_from_file_location("_vgpack", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _pack = mod
    return _pack


def lib():
    """The loaded library (raises NativeUnavailable if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; "
            f"g.build()\"` (nvcc, sm_100a). There is no CPU fallback.")
    try:
        handle = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:  # pragma: no cover - depends on the host
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (restype, argtypes) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if handle.vg_abi_version() != ABI_VERSION:
        raise NativeUnavailable(f"ABI mismatch: library {handle.vg_abi_version()} != {ABI_VERSION}")
    _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc != VG_OK:
        msg = lib().vg_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")
