"""B200-native parallel uniform-grid build (arXiv 2403.10647, Alg. 1 BuildParallelGrid).

Drop-in for the reference's hot path `pargrid.builders.build_parallel` (builders.py:144):
host code here, sm_100a CUDA kernels behind the C ABI in include/pgrid.h.
"""

from .errors import DeviceError, GridError, InvariantError, ObjParseError, SizeError
from .gridcore import (Aabb, CompactGrid, GridSpec, TriangleMesh, compute_dims, grids_equal,
                       mesh_bounds, spec_for_mesh)
from .scenes import gen_scene
from .builders import PHASES, BuildReport, build_compact, build_parallel, build_sorted
from .stats import GridStats, compute_stats, estimate_pairs, grid_memory_bytes
from .traverse import Hit, Ray, RayCaster, dda_cast, dda_traverse

__version__ = "0.1.0"

__all__ = ["Aabb", "BuildReport", "CompactGrid", "DeviceError", "GridError", "GridSpec", "GridStats", "Hit",
           "Ray", "RayCaster", "compute_stats", "dda_cast", "dda_traverse", "estimate_pairs", "grid_memory_bytes",
           "InvariantError", "ObjParseError", "PHASES", "SizeError", "TriangleMesh",
           "build_compact", "build_parallel", "build_sorted", "compute_dims", "gen_scene", "grids_equal", "mesh_bounds",
           "spec_for_mesh"]
