"""B200-native batched point-in-convex-polygon engine (arxiv 2007.15385).

The product is libvpipg.so (CUDA kernels for sm_100a + the C-ABI in
include/vpipg.h + the vpip:: C++ API in include/vpip/). This package holds its
sources (csrc/), the build recipe and a thin Python host mirror over ctypes.
"""
from ._lib import LIB_PATH, VpipError, load  # noqa: F401
from .engine import (F32, F64, KIND_ALL, KIND_CROSSING, KIND_OFFSET, KIND_VORONOI,  # noqa: F401
                     PolygonDB, PreparedPolygon, fill_join_pairs, fill_uniform_points, mix_seed,
                     random_convex_polygon, regular_polygon, release_staging, sample_points,
                     zero_counts)
