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
