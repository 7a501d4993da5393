"""`GpuOctree`: the reference's `Octree` (model.py:170-196) backed by a device tree.

The node hierarchy, leaf points and voxels live in HBM (`DeviceTree`).  The
Python `OctreeNode` objects are materialised lazily on first access to `.root`,
with exactly the reference's fields: octant `path`, `bounds` (fp64 sequential
child_bounds fold, computed on the device), `children` (8 slots, None = absent),
leaf `point_positions` (float64, input order) / `point_colors`, inner
`voxel_coords` / `voxel_colors` (uint8, in the reference's stored order: ascending
x-major key, or winning ordinal for first-come) and `oversized`.
`build_lod` on a materialised tree updates the inner nodes in place, like the
reference (sampling.py:172-176).
"""
from __future__ import annotations

import numpy as np

from .device import DeviceTree, unpack_records
from .model import AABB, BuildConfig, Octree, OctreeNode


def cell_path(cell, depth: int) -> tuple[int, ...]:
    cx, cy, cz = (int(c) for c in cell)
    return tuple(((cx >> b) & 1) | (((cy >> b) & 1) << 1) | (((cz >> b) & 1) << 2)
                 for b in range(depth - 1, -1, -1))


def decode_voxels(raw: np.ndarray):
    """(m, 2) u32 {key, rgb} -> coords (m,3) u8, colors (m,3) u8."""
    key = raw[:, 0]
    rgb = raw[:, 1]
    coords = np.stack([key >> 14, (key >> 7) & 127, key & 127], axis=1).astype(np.uint8)
    colors = np.stack([rgb & 255, (rgb >> 8) & 255, (rgb >> 16) & 255], axis=1).astype(np.uint8)
    return coords, colors


class GpuOctree(Octree):
    """Octree whose storage is a `DeviceTree`; Python nodes are built on demand."""

    def __init__(self, dev: DeviceTree, config: BuildConfig):
        self._dev = dev
        self._generation = dev.generation
        self.config = config
        info = dev.info()
        self.world_bounds = AABB(tuple(float(v) for v in info.world_min), float(info.world_size))
        self._root = None
        self._nodes = None       # node table (numpy structured)
        self._objs = None        # node id -> OctreeNode
        self.strategy_built = None

    def _check_live(self):
        """A DeviceTree's buffers are reused by its next split: a tree built earlier on the same
        handle must not silently show the new build's data."""
        if self._dev.generation != self._generation:
            raise RuntimeError("this tree's device buffers were reused by a later build on the same DeviceTree; "
                               "materialise it (tree.root) before reusing the handle, or use a new DeviceTree")

    @property
    def device_tree(self) -> DeviceTree:
        self._check_live()
        return self._dev

    @property
    def root(self) -> OctreeNode:
        if self._root is None:
            self._check_live()
            self._materialize()
        return self._root

    def _materialize(self):
        nodes = self._dev.nodes()
        pos, col = unpack_records(self._dev.leaf_records(), self._dev.info().point_format)
        objs = []
        for k in range(len(nodes)):
            nd = nodes[k]
            depth = int(nd["depth"])
            path = cell_path(nd["cell"], depth)
            b = AABB((float(nd["min"][0]), float(nd["min"][1]), float(nd["min"][2])), float(nd["size"]))
            if nd["flags"] & 1:
                f, c = int(nd["first"]), int(nd["count"])
                obj = OctreeNode(path, b, None, pos[f:f + c], col[f:f + c], oversized=bool(nd["flags"] & 2))
            else:
                obj = OctreeNode(path, b, children=[None] * 8)
            objs.append(obj)
        for k in range(len(nodes)):
            if objs[k].children is not None:
                for o, c in enumerate(nodes[k]["child"]):
                    if c >= 0:
                        objs[k].children[o] = objs[int(c)]
        self._nodes = nodes
        self._objs = objs
        self._root = objs[0]
        if self._dev.info().voxel_mode >= 0:
            self._refresh_voxels()

    def _refresh_voxels(self):
        """Copy the device voxels into the inner OctreeNode objects (in place)."""
        if self._objs is None:
            return
        nodes = self._dev.nodes()
        coords, colors = decode_voxels(self._dev.voxels())
        for k in range(len(nodes)):
            if nodes[k]["flags"] & 1:
                continue
            f, c = int(nodes[k]["first"]), int(nodes[k]["count"])
            self._objs[k].voxel_coords = coords[f:f + c]
            self._objs[k].voxel_colors = colors[f:f + c]

    # cheap summaries straight from the node table (no materialisation)
    @property
    def node_count(self) -> int:
        if self._objs is not None:
            return len(self._objs)
        self._check_live()
        return int(self._dev.info().n_nodes)

    @property
    def point_count(self) -> int:
        if self._objs is not None:
            return sum(len(o.point_positions) for o in self._objs if o.children is None)
        self._check_live()
        return int(self._dev.info().n_points)
