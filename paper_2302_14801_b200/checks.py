"""Structural invariant checks (reference checks.py:1-96), evaluated on the device for
trees built here: `lod_tree_checks` returns one byte of failure bits per node; the host
turns them into the reference's `CheckResult` list (same names, order and details --
offending paths in DFS preorder, first five).  Trees that exist only as host objects
(e.g. from `codec.decode`) are checked with the same rules in numpy."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .model import GRID_SIZE, Octree

CAPACITY, OVERSIZED, MAXIMALITY, CONTAINMENT, VOXEL_BOUNDS, UNIQUENESS, EMPTY_INNER, NO_CHILDREN = (
    1, 2, 4, 8, 16, 32, 64, 128)   # include/lodb200.h lod_check_bit


@dataclass
class CheckResult:
    name: str
    passed: bool
    detail: str = ""


def _results(total, expected, bad, require_lod):
    """Assemble the reference's result list from offending-path lists (checks.py:24-92)."""
    if expected is None:
        expected = total
    r = [CheckResult("conservation", total == expected, f"leaf points {total}, expected {expected}"),
         CheckResult("capacity", not bad[CAPACITY], f"overfull leaves: {bad[CAPACITY][:5]}"),
         CheckResult("oversized-at-max-depth", not bad[OVERSIZED], f"misplaced oversized: {bad[OVERSIZED][:5]}"),
         CheckResult("merging-maximality", not bad[MAXIMALITY], f"undersized inner nodes: {bad[MAXIMALITY][:5]}"),
         CheckResult("containment", not bad[CONTAINMENT], f"out-of-bounds leaves: {bad[CONTAINMENT][:5]}"),
         CheckResult("voxel-bounds", not bad[VOXEL_BOUNDS], f"out-of-range voxels: {bad[VOXEL_BOUNDS][:5]}"),
         CheckResult("voxel-uniqueness", not bad[UNIQUENESS], f"duplicate voxels: {bad[UNIQUENESS][:5]}")]
    if require_lod:
        r.append(CheckResult("inner-non-empty", not bad[EMPTY_INNER], f"empty inner nodes: {bad[EMPTY_INNER][:5]}"))
    r.append(CheckResult("inner-has-children", not bad[NO_CHILDREN], f"childless inner nodes: {bad[NO_CHILDREN][:5]}"))
    return r


def _device_checks(tree, expected_points, require_lod):
    import torch
    from .codec import path_sort_keys
    from .octree import cell_path
    dev = tree.device_tree
    nodes = dev.nodes()
    flags = np.zeros(len(nodes), np.uint8)
    _abi.check(dev.lib.lod_tree_checks(dev.h, int(tree.config.T), int(tree.config.max_depth),
                                       flags.ctypes.data_as(C.c_void_p),
                                       C.c_void_p(torch.cuda.current_stream(dev.device).cuda_stream)))
    order = np.argsort(path_sort_keys(nodes["cell"], nodes["depth"]), kind="stable")   # DFS preorder
    bad = {}
    for bit in (CAPACITY, OVERSIZED, MAXIMALITY, CONTAINMENT, VOXEL_BOUNDS, UNIQUENESS, EMPTY_INNER, NO_CHILDREN):
        hit = order[(flags[order] & bit) != 0]
        bad[bit] = [cell_path(nodes[k]["cell"], int(nodes[k]["depth"])) for k in hit[:5]] + \
            [None] * max(0, int(len(hit)) - 5)   # only the first five are printed
    leaf = (nodes["flags"] & 1).astype(bool)
    total = int(nodes["count"][leaf].sum())
    return _results(total, expected_points, bad, require_lod)


def _host_checks(tree: Octree, expected_points, require_lod):
    cfg = tree.config
    leaves, inner = tree.leaves(), tree.inner_nodes()
    bad = {b: [] for b in (CAPACITY, OVERSIZED, MAXIMALITY, CONTAINMENT, VOXEL_BOUNDS, UNIQUENESS, EMPTY_INNER,
                           NO_CHILDREN)}
    for n in leaves:
        if not n.oversized and n.point_count > cfg.T:
            bad[CAPACITY].append(n.path)
        if n.oversized and n.depth != cfg.max_depth:
            bad[OVERSIZED].append(n.path)
        if n.point_count == 0:
            bad[CONTAINMENT].append(n.path)
            continue
        tol = n.bounds.size * 1e-6
        rel = n.point_positions - n.bounds.min_array()
        if (rel < -tol).any() or (rel > n.bounds.size + tol).any():
            bad[CONTAINMENT].append(n.path)
    for node in inner:
        kids = [c for _, c in node.existing_children()]
        if kids and all(k.is_leaf for k in kids) and sum(k.point_count for k in kids) < cfg.T:
            bad[MAXIMALITY].append(node.path)
        if not kids:
            bad[NO_CHILDREN].append(node.path)
        if node.voxel_count == 0:
            bad[EMPTY_INNER].append(node.path)
            continue
        c = node.voxel_coords.astype(np.int64)
        if (c < 0).any() or (c >= GRID_SIZE).any():
            bad[VOXEL_BOUNDS].append(node.path)
        keys = (c[:, 0] * GRID_SIZE + c[:, 1]) * GRID_SIZE + c[:, 2]
        if len(np.unique(keys)) != len(keys):
            bad[UNIQUENESS].append(node.path)
    return _results(sum(n.point_count for n in leaves), expected_points, bad, require_lod)


def run_checks(tree: Octree, expected_points: int | None = None, require_lod: bool = True) -> list[CheckResult]:
    """checks.py:18-92."""
    from .octree import GpuOctree
    if isinstance(tree, GpuOctree):
        return _device_checks(tree, expected_points, require_lod)
    return _host_checks(tree, expected_points, require_lod)


def all_passed(results: list[CheckResult]) -> bool:
    return all(r.passed for r in results)
