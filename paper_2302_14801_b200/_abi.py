"""ctypes binding of `include/lodb200.h` (the in-tree `_lib/liblodb200.so`).

There is no CPU fallback: if the library or a CUDA device is missing, the
product API raises.  Status codes map to the reference's exceptions
(`include/lodb200.h`): 1 ValueError, 2 ConsistencyError, 3 RuntimeError,
4 NotImplementedError.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import ConsistencyError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "liblodb200.so")

LOD_POINTS_F32, LOD_POINTS_F64 = 0, 1
LOD_MODE_RANDOM, LOD_MODE_AVERAGE, LOD_MODE_FIRST_COME, LOD_MODE_WEIGHTED = 0, 1, 2, 3


class LodConfig(C.Structure):
    _fields_ = [("T", C.c_uint32), ("initial_depth", C.c_int32), ("extension_depth", C.c_int32),
                ("max_depth", C.c_int32)]


class LodTreeInfo(C.Structure):
    _fields_ = [("n_points", C.c_uint64), ("n_voxels", C.c_uint64), ("n_nodes", C.c_uint32),
                ("n_leaves", C.c_uint32), ("n_inner", C.c_uint32), ("depth", C.c_uint32),
                ("point_format", C.c_int32), ("voxel_mode", C.c_int32), ("world_min", C.c_double * 3),
                ("world_size", C.c_double), ("n_ext_grids", C.c_uint32), ("radix_passes", C.c_uint32)]


class LodNode(C.Structure):
    _fields_ = [("min", C.c_double * 3), ("size", C.c_double), ("first", C.c_uint64), ("count", C.c_uint32),
                ("parent", C.c_int32), ("cell", C.c_uint16 * 3), ("depth", C.c_uint8), ("flags", C.c_uint8),
                ("child", C.c_int32 * 8)]


class LodExtGrid(C.Structure):
    _fields_ = [("pyr_off", C.c_uint64), ("ax", C.c_uint16), ("ay", C.c_uint16), ("az", C.c_uint16),
                ("base", C.c_uint8), ("ext", C.c_uint8)]


class LodSpan(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("n", C.c_uint64)]


# numpy view of lod_node (88 bytes)
NODE_DTYPE = None


def node_dtype():
    global NODE_DTYPE
    if NODE_DTYPE is None:
        import numpy as np
        NODE_DTYPE = np.dtype([("min", "<f8", 3), ("size", "<f8"), ("first", "<u8"), ("count", "<u4"),
                               ("parent", "<i4"), ("cell", "<u2", 3), ("depth", "u1"), ("flags", "u1"),
                               ("child", "<i4", 8)])
        assert NODE_DTYPE.itemsize == C.sizeof(LodNode) == 88
    return NODE_DTYPE


# (name, restype, argtypes) of every exported symbol -- mirrors include/lodb200.h
_P = C.c_void_p
SIGNATURES = [
    ("lod_tree_create", _P, [C.c_int]),
    ("lod_tree_destroy", None, [_P]),
    ("lod_split", C.c_int, [_P, _P, C.c_uint64, C.c_int, C.POINTER(C.c_double), C.POINTER(LodConfig), _P]),
    ("lod_voxelize", C.c_int, [_P, C.c_int, C.c_uint64, _P]),
    ("lod_build", C.c_int, [_P, _P, C.c_uint64, C.c_int, C.POINTER(LodConfig), C.c_int, C.c_uint64, _P]),
    ("lod_tree_get_info", C.c_int, [_P, C.POINTER(LodTreeInfo)]),
    ("lod_tree_copy_nodes", C.c_int, [_P, _P, _P]),
    ("lod_tree_leaf_points", C.c_int, [_P, C.POINTER(C.c_void_p)]),
    ("lod_tree_voxels", C.c_int, [_P, C.POINTER(C.c_void_p)]),
    ("lod_tree_copy_leaf_points", C.c_int, [_P, _P, _P]),
    ("lod_tree_copy_voxels", C.c_int, [_P, _P, _P]),
    ("lod_tree_copy_async", C.c_int, [_P, _P, _P, _P, _P]),
    ("lod_tree_copy_range", C.c_int, [_P, C.c_int, C.c_uint64, C.c_uint64, _P, _P]),
    ("lod_tree_encode_payload", C.c_int, [_P, _P, _P, C.c_uint32, _P, _P]),
    ("lod_ingest_las", C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_int32, _P, _P, _P, _P]),
    ("lod_ingest_ply", C.c_int, [_P, C.c_uint64, C.c_uint32, _P, _P, C.c_int, C.c_int, _P, _P]),
    ("lod_tree_checks", C.c_int, [_P, C.c_uint32, C.c_int32, _P, _P]),
    ("lod_tree_device_bytes", C.c_uint64, [_P]),
    ("lod_set_allocator", C.c_int, [_P, _P, _P]),
    ("lod_workspace_bytes", C.c_int, [C.c_uint64, C.c_int, C.POINTER(LodConfig), C.c_int, C.POINTER(C.c_uint64)]),
    ("lod_set_timing", C.c_int, [_P, C.c_int]),
    ("lod_tree_stage_ms", C.c_int, [_P, C.POINTER(C.c_float)]),
    ("lod_tree_kernel_ms", C.c_int, [_P, C.POINTER(C.c_float)]),
    ("lod_tree_launches", C.c_uint64, [_P]),
    ("lod_pack_points", C.c_int, [_P, C.c_int, _P, C.c_uint64, C.c_int, _P, C.POINTER(C.c_int), _P]),
    ("lod_tree_set_output_wait", C.c_int, [_P, _P]),
    ("lod_dist_leaf_buffer", C.c_int, [_P, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("lod_merge_pyramid", C.c_int, [_P, C.c_int, C.c_uint32, _P]),
    ("lod_tree_copy_point_keys", C.c_int, [_P, _P, _P]),
    ("lod_tree_copy_pyramids", C.c_int, [_P, _P, C.POINTER(C.c_uint64), _P]),
    ("lod_tree_ext_grids", C.c_int, [_P, _P, C.POINTER(C.c_uint32), _P]),
    ("lod_tree_ext_points", C.c_int, [_P, _P, _P, C.POINTER(C.c_uint64), _P]),
    ("lod_project_samples", C.c_int, [C.c_int, _P, C.c_uint64, C.POINTER(C.c_double), C.c_double, C.c_int, _P, _P]),
    ("lod_extract", C.c_int, [C.c_int, _P, _P, C.c_uint64, C.c_uint64, C.c_uint64, _P, _P, C.POINTER(C.c_uint64),
                              _P]),
    ("lod_generate", C.c_int, [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64, _P, C.POINTER(C.c_double), _P]),
    ("lod_dist_begin", C.c_int, [_P, _P, C.c_uint64, C.c_int, C.POINTER(LodConfig), _P, _P]),
    ("lod_dist_count", C.c_int, [_P, C.c_uint64, _P, C.POINTER(LodSpan), _P]),
    ("lod_dist_extend", C.c_int, [_P, C.POINTER(LodSpan), _P]),
    ("lod_dist_skeleton", C.c_int, [_P, _P, _P]),
    ("lod_dist_leaf_counts", C.c_int, [_P, _P]),
    ("lod_dist_copy_segments", C.c_int, [_P, _P, _P, _P, _P, _P, C.c_uint64, _P]),
    ("lod_dist_adopt", C.c_int, [_P, _P, C.c_uint64, _P, _P]),
    ("lod_dist_voxelize", C.c_int, [_P, C.c_int, C.c_uint64, _P, C.c_int, _P, _P, C.c_uint32, C.c_uint32, _P,
                                    _P]),
    ("lod_dist_export_roots", C.c_int, [_P, _P, C.c_uint32, _P, _P, _P]),
    ("lod_comm_unique_id", C.c_int, [_P]),
    ("lod_comm_init", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("lod_comm_destroy", C.c_int, [_P]),
    ("lod_comm_allreduce", C.c_int, [_P, _P, C.c_uint64, C.c_int, C.c_int, _P]),
    ("lod_comm_allgather", C.c_int, [_P, _P, _P, C.c_uint64, _P]),
    ("lod_comm_alltoallv", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("lod_comm_gatherv", C.c_int, [_P, _P, C.c_uint64, _P, _P, C.c_int, _P]),
    ("lod_last_error", C.c_char_p, []),
    ("lod_version", C.c_char_p, []),
]

_lib = None


def load(build_if_missing: bool = False) -> C.CDLL:
    """Load the CUDA library; raise loudly if it is not built (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2302_14801_b200.build` "
                "(the LOD path has no CPU fallback)")
        from .build import build
        build()
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code: int) -> None:
    if code == 0:
        return
    msg = (load().lod_last_error() or b"").decode()
    if code == 1:
        raise ValueError(msg)
    if code == 2:
        raise ConsistencyError(msg)
    if code == 4:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)
