"""B200-native tilemesh hot path: tiled MFIter stencil sweeps + FillBoundary.

Drop-in for the reference package ``tilemesh``
(/root/reference/pkg/src/tilemesh/__init__.py) on the hot path: the same
names (Box algebra, BoxArray, Geometry, MultiFab, build_fill_plan,
fill_boundary, build_schedule, TileCursor, HeatParams, heat_step) plus the
north-star additions DistributionMapping, MFIter, FillBoundary, the GSRB /
residual kernels and the wide4 (8th-order, 4-ghost) step.  Storage lives on
the GPU; every data-path operation is an sm_100a kernel of
libtilemesh_b200.so (no CPU fallback).
"""

from .box import Box, box_diff, decompose, grow, intersect, shift, to_face
from .boxarray import BoxArray, DistributionMapping, Geometry, partition
from .configs import CONFIGS, Workload, make_init
from .fab import FArrayBox, copy_region, intersect_copy
from .fillplan import CopyTag, FillPlan, build_fill_plan, shift_candidates, split_tags
from .mfiter import (
    DEFAULT_TILE_SIZE,
    MFIter,
    TileCursor,
    TileSchedule,
    build_schedule,
    parallel_for_tiles,
)
from .multifab import CONTIGUOUS, REGIONAL, DeviceFab, FillBoundary, MultiFab, fill_boundary
from .plotfile import read_plotfile, write_plotfile
from .stencil import (
    HeatParams,
    gsrb_color,
    gsrb_solve,
    gsrb_sweep,
    heat_amplification,
    heat_divergence_update,
    heat_flux,
    heat_step,
    init_cosine,
    residual_maxnorm,
)
from .wide4 import (
    StencilCoeffs8,
    Wide4Runner,
    derive_coeffs8,
    wide4_amplification,
    wide4_stable_dt,
    wide4_step,
)

__all__ = [
    "Box", "box_diff", "decompose", "grow", "intersect", "shift", "to_face",
    "BoxArray", "DistributionMapping", "Geometry", "partition",
    "CONFIGS", "Workload", "make_init", "FArrayBox", "copy_region", "intersect_copy",
    "CopyTag", "FillPlan", "build_fill_plan", "shift_candidates", "split_tags",
    "DEFAULT_TILE_SIZE", "MFIter", "TileCursor", "TileSchedule", "build_schedule", "parallel_for_tiles",
    "CONTIGUOUS", "REGIONAL", "DeviceFab", "FillBoundary", "MultiFab", "fill_boundary",
    "read_plotfile", "write_plotfile",
    "HeatParams", "gsrb_color", "gsrb_solve", "gsrb_sweep", "heat_amplification", "heat_divergence_update", "heat_flux", "heat_step", "init_cosine",
    "residual_maxnorm",
    "StencilCoeffs8", "Wide4Runner", "derive_coeffs8", "wide4_amplification", "wide4_stable_dt",
    "wide4_step",
]

__version__ = "0.1.0"
