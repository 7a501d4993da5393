"""paper_2302_14801_b200: B200-native LOD construction for colored point clouds.

Drop-in for the reference's construction path (`lodforge.partition.partition` +
`lodforge.sampling.build_lod`, all four strategies: first-come, random, average ==
color_filter, weighted) and its VLPC file format (`lodforge.codec`), running as
hand-written sm_100a CUDA kernels behind a C ABI (`include/lodb200.h`).
"""
from . import checks, codec, ingest
from .errors import ConsistencyError, FormatError
from .model import (AABB, GRID_SIZE, STRATEGIES, BuildConfig, ColorRGB, Octree, OctreeNode, Point, PointCloud,
                    bounds_at, cell_of, cells_of, child_bounds, world_bounds_of)
from .partition import Partitioner, partition
from .sampling import build_lod, build_lod_points

__all__ = [
    "AABB", "BuildConfig", "ColorRGB", "ConsistencyError", "FormatError", "GRID_SIZE", "Octree", "OctreeNode",
    "Point", "PointCloud", "Partitioner", "STRATEGIES", "bounds_at", "build_lod", "build_lod_points", "cell_of",
    "cells_of", "checks", "child_bounds", "codec", "ingest", "partition", "world_bounds_of",
]

__version__ = "0.1.0"
