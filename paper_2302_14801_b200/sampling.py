"""Drop-in for `lodforge.sampling.build_lod` (reference sampling.py:165-176) on the B200,
plus the north-star fused entry point.

    build_lod(tree, strategy=None, seed=None) -> tree          # reference form
    build_lod(points, colors, T=50_000, grid=128, mode="color_filter", seed=0)  # fused

All four reference strategies run on the GPU: "first-come" (the reference default,
model.py:115), "random", "average" (alias "color_filter") and "weighted" (colours
within +-1 per channel of the reference's fp64 sums, SPEC.md).  There is no CPU
fallback; unknown names raise ValueError like the reference (sampling.py:169-170).
"""
from __future__ import annotations

import dataclasses

import numpy as np

from ._abi import LOD_MODE_AVERAGE, LOD_MODE_FIRST_COME, LOD_MODE_RANDOM, LOD_MODE_WEIGHTED
from .device import DeviceTree, make_config
from .model import GRID_SIZE, MODE_ALIASES, BuildConfig, Octree
from .octree import GpuOctree

MAX_RANDOM_SAMPLES = 1 << 20  # reference sampling.py:18


_CODES = {"random": LOD_MODE_RANDOM, "average": LOD_MODE_AVERAGE, "first-come": LOD_MODE_FIRST_COME,
          "weighted": LOD_MODE_WEIGHTED}


def _mode_code(strategy: str) -> int:
    if strategy in MODE_ALIASES:
        return _CODES[MODE_ALIASES[strategy]]
    raise ValueError(f"unknown sampling strategy: {strategy}")


def build_lod(tree_or_points, strategy_or_colors=None, seed=None, **kw):
    """Fill inner nodes with voxels, deepest first.  See module docstring for both forms."""
    if isinstance(tree_or_points, Octree):
        if kw:
            raise TypeError(f"unexpected keyword arguments {sorted(kw)}")
        return _build_tree(tree_or_points, strategy_or_colors, seed)
    return build_lod_points(tree_or_points, strategy_or_colors, seed=0 if seed is None else seed, **kw)


def _build_tree(tree: Octree, strategy: str | None, seed: int | None) -> Octree:
    strategy = tree.config.strategy if strategy is None else strategy
    seed = tree.config.seed if seed is None else seed
    code = _mode_code(strategy)
    if not isinstance(tree, GpuOctree):
        raise TypeError("build_lod needs a tree produced by paper_2302_14801_b200.partition")
    tree.device_tree.voxelize(code, seed)
    tree.strategy_built = strategy
    tree._refresh_voxels()
    return tree


def build_lod_points(points, colors, T: int = 50_000, grid: int = GRID_SIZE, mode: str = "color_filter",
                     seed: int = 0, device_tree: DeviceTree | None = None, config: BuildConfig | None = None):
    """North-star fused form: split + voxelize in one call, world bounds from the points.

    `points` (n,3) float32/float64 and `colors` (n,3) uint8 host arrays.  `grid` must be
    128 (the reference's fixed GRID_SIZE, model.py:18).
    """
    if grid != GRID_SIZE:
        raise ValueError(f"grid must be {GRID_SIZE} (the reference's fixed sampling grid)")
    code = _mode_code(mode)
    pos = np.asarray(points)
    if pos.ndim != 2 or pos.shape[1] != 3:
        pos = pos.reshape(-1, 3)
    if len(pos) == 0:
        raise ValueError("cannot partition an empty point cloud")
    if config is None:
        cfg = BuildConfig(T=T, strategy=MODE_ALIASES[mode], seed=seed)
    else:
        if T != 50_000 and T != config.T:
            raise ValueError(f"T={T} conflicts with config.T={config.T}")
        # the tree's config records what was actually built (codec.encode writes it)
        cfg = dataclasses.replace(config, strategy=MODE_ALIASES[mode], seed=seed)
    dev = device_tree or DeviceTree()
    d_rec, fmt, n = dev.upload(pos, colors)
    dev.build(d_rec, n, fmt, make_config(cfg.T, cfg.initial_depth, cfg.extension_depth, cfg.max_depth), code, seed)
    tree = GpuOctree(dev, cfg)
    tree.strategy_built = MODE_ALIASES[mode]
    return tree


# ---------------------------------------------------------------------------
# The reference's per-node helpers (sampling.py:21-162) on the device, for callers driving
# the stages themselves: lod_project_samples / lod_extract (csrc/extract.cu).
# ---------------------------------------------------------------------------

def _torch_dev():
    from .device import _torch
    return _torch()


def _stream():
    from .device import current_stream_ptr
    return current_stream_ptr()


def project_child_samples(node):
    """All child samples of an inner node in its 128^3 grid, canonical ordinal order
    (children in octant order, each child's samples in stored order): (S,3) float64 grid
    positions and (S,3) uint8 colours (reference sampling.py:21-47)."""
    import ctypes as C
    from . import _abi
    from .errors import ConsistencyError
    torch = _torch_dev()
    if node.is_leaf:
        raise ValueError("cannot project samples for a leaf node")
    lib = _abi.load()
    mn = (C.c_double * 3)(*[float(v) for v in node.bounds.min])
    parts, cols = [], []
    for octant, child in node.existing_children():
        if child.sample_count == 0:
            raise ConsistencyError(f"child {child.path} has no samples")
        if child.is_leaf:
            src = torch.from_numpy(np.ascontiguousarray(child.point_positions, np.float64)).cuda()
            kind, col = 0, child.point_colors
        else:
            src = torch.from_numpy(np.ascontiguousarray(child.voxel_coords, np.uint8)).cuda()
            kind, col = 1, child.voxel_colors
        n = len(col)
        out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        _abi.check(lib.lod_project_samples(kind, C.c_void_p(src.data_ptr()), n, mn, float(node.bounds.size), octant,
                                           C.c_void_p(out.data_ptr()), _stream()))
        parts.append(out)
        cols.append(np.asarray(col, np.uint8))
    return torch.cat(parts).cpu().numpy(), np.concatenate(cols)


def _extract(code, gpos, colors, seed=0, node_hash=0):
    import ctypes as C
    from . import _abi
    torch = _torch_dev()
    g = np.ascontiguousarray(gpos, np.float64).reshape(-1, 3)
    c = np.ascontiguousarray(colors, np.uint8).reshape(-1, 3)
    if len(g) != len(c):
        raise ValueError("positions/colors length mismatch")
    S = len(g)
    dg = torch.from_numpy(g).cuda()
    dc = torch.from_numpy(c).cuda()
    oc = torch.empty((max(S, 1), 3), dtype=torch.uint8, device="cuda")
    ok = torch.empty((max(S, 1), 3), dtype=torch.uint8, device="cuda")
    m = C.c_uint64(0)
    _abi.check(_abi.load().lod_extract(code, C.c_void_p(dg.data_ptr()), C.c_void_p(dc.data_ptr()), S,
                                       int(seed) & ((1 << 64) - 1), int(node_hash) & ((1 << 64) - 1),
                                       C.c_void_p(oc.data_ptr()), C.c_void_p(ok.data_ptr()), C.byref(m), _stream()))
    m = int(m.value)
    return oc[:m].cpu().numpy(), ok[:m].cpu().numpy()


def extract_first_come(gpos, colors):
    """Per cell the smallest ordinal wins; voxels listed by winning ordinal (sampling.py:61-66)."""
    return _extract(LOD_MODE_FIRST_COME, gpos, colors)


def extract_random(gpos, colors, seed: int, node_hash: int):
    """Per cell the largest (rand12 | ordinal20) wins; ascending cell key (sampling.py:69-85)."""
    return _extract(LOD_MODE_RANDOM, gpos, colors, seed, node_hash)


def extract_average(gpos, colors):
    """Per cell the rounded mean colour (half away from zero); ascending key (sampling.py:88-97)."""
    return _extract(LOD_MODE_AVERAGE, gpos, colors)


def extract_weighted(gpos, colors):
    """Distance-weighted 2x2x2 mean, occupied cells only (sampling.py:100-133); colours within
    +-1 of the reference's sequential fp64 sums (exact 2^-24 fixed point here)."""
    return _extract(LOD_MODE_WEIGHTED, gpos, colors)


def _sample_node(node, strategy: str, seed: int):
    from . import rng
    gpos, colors = project_child_samples(node)
    if strategy == "first-come":
        return extract_first_come(gpos, colors)
    if strategy == "random":
        return extract_random(gpos, colors, seed, rng.path_hash(seed, node.path))
    if strategy == "average":
        return extract_average(gpos, colors)
    if strategy == "weighted":
        return extract_weighted(gpos, colors)
    raise ValueError(f"unknown sampling strategy: {strategy}")


def sample_first_come(node):
    return _sample_node(node, "first-come", 0)


def sample_random(node, seed: int):
    return _sample_node(node, "random", seed)


def sample_average(node):
    return _sample_node(node, "average", 0)


def sample_weighted(node):
    return _sample_node(node, "weighted", 0)
