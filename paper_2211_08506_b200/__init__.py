"""voxgrid-b200: B200-native batched molecule -> Gaussian-density grid generation.

Drop-in for the grid-generation path of the reference package ``voxgrid``
(ParticleGrid, arXiv 2211.08506): same names and arguments, device-resident
float32 grids ``(B, C, H, W, D)`` computed by hand-written sm_100a kernels.
See DESIGN.md for the boundary and INTEGRATION.md for the C-ABI.
"""

from .core import (
    BoundingBox,
    Grid,
    GridSpec,
    LatticeCell,
    ParticleSet,
    bounding_box_of,
    voxel_to_world,
    world_to_voxel,
)
from .gridgen import (
    BatchResult,
    GenStats,
    GridEngine,
    check_packed,
    default_engine,
    flagged_molecules,
    generate_batch,
    generate_grid,
    generate_packed,
)
from .kernels import ERF_C1, ERF_C2, AxisTable, axis_tables_batch, erf_approx, fused_axis_tables
from .io import (
    ELEMENT_SYMBOLS,
    MoleculeFile,
    ParseError,
    grid_from_array,
    pack_molecules,
    parse_points_csv,
    parse_xyz,
    read_npy,
    write_npy,
)
from .loader import GridPipeline
from .reversal import (
    CountMismatchWarning,
    Peak,
    PeakSet,
    ReversalConfig,
    ReversalState,
    detect_peaks,
    loss,
    loss_gradient,
    refine_coords,
    refine_coords_batch,
    reverse_grid,
    reverse_grids,
)
from .cli import cli_main

__version__ = "0.1.0"


def __getattr__(name):
    # deferred like the reference (__init__.py:59-65): sklearn only when asked
    if name == "GaussianVoxelizer":
        from .estimator import GaussianVoxelizer

        return GaussianVoxelizer
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


__all__ = [
    "BoundingBox",
    "Grid",
    "GridSpec",
    "LatticeCell",
    "ParticleSet",
    "bounding_box_of",
    "voxel_to_world",
    "world_to_voxel",
    "BatchResult",
    "GenStats",
    "GridEngine",
    "default_engine",
    "generate_batch",
    "generate_grid",
    "generate_packed",
    "check_packed",
    "flagged_molecules",
    "ERF_C1",
    "ERF_C2",
    "AxisTable",
    "axis_tables_batch",
    "erf_approx",
    "fused_axis_tables",
    "GaussianVoxelizer",
    "ELEMENT_SYMBOLS",
    "MoleculeFile",
    "ParseError",
    "grid_from_array",
    "pack_molecules",
    "parse_points_csv",
    "parse_xyz",
    "read_npy",
    "write_npy",
    "GridPipeline",
    "CountMismatchWarning",
    "Peak",
    "PeakSet",
    "ReversalConfig",
    "ReversalState",
    "detect_peaks",
    "loss",
    "loss_gradient",
    "refine_coords",
    "refine_coords_batch",
    "reverse_grid",
    "reverse_grids",
    "cli_main",
    "__version__",
]
