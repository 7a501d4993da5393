"""Drop-in for `lodforge.partition` (reference partition.py:79-302) on the B200.

`partition(cloud, config)` and `Partitioner(cloud, config, bounds).run()` keep the
reference's signatures, defaults and exceptions; the hierarchical counting sort runs
in `liblodb200.so` (count -> extension rounds -> merge pyramid -> node table ->
stable distribute).  The result is a `GpuOctree`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .device import DeviceTree, make_config
from .errors import ConsistencyError
from .model import AABB, BuildConfig, Octree, PointCloud
from .octree import GpuOctree, cell_path

UNMERGEABLE = 0xFFFFFFFF  # reference partition.py:20


@dataclass
class ExtendedPyramid:
    """Sub-pyramid refining one overfull cell (reference partition.py:64-76), read back from the
    device build: the grid's counts, its member points and their cells in its finest grid."""

    anchor_path: tuple[int, ...]
    anchor_cell: np.ndarray  # absolute grid coords of the anchor at its level
    depth: int  # number of extra levels (finest grid is (2^depth)^3)
    finest: np.ndarray
    point_idx: np.ndarray  # global indices of the anchor's points, input order
    rel_cells: np.ndarray  # (n, 3) finest-level coords relative to the anchor
    children: dict[tuple[int, int, int], "ExtendedPyramid"] = field(default_factory=dict)
    levels: list[np.ndarray] | None = None  # filled by merge
    refs: list[np.ndarray] | None = None  # per-level leaf-id grids, filled by build_targets


def merge_pyramid(finest: np.ndarray, T: int) -> list[np.ndarray]:
    """Merge a counting grid bottom-up into a full pyramid on the device (partition.py:36-61).

    A 2x2x2 group of plain counters summing below T is replaced by its sum one level up and
    zeroed; a group at or above T, or containing an UNMERGEABLE cell, flags the parent
    UNMERGEABLE.  Returns int64 grids from the 1^3 root (index 0) down to the input grid.
    """
    import torch
    from . import _abi
    from .device import current_stream_ptr
    finest = np.asarray(finest)
    dim = finest.shape[0] if finest.ndim == 3 else 0
    if finest.ndim != 3 or finest.shape != (dim, dim, dim) or dim & (dim - 1) or dim > 1024:
        raise ValueError("finest must be a (2^L)^3 grid with L <= 10")
    if ((finest < 0) | (finest > UNMERGEABLE)).any():
        raise ValueError("counts must lie in [0, 0xFFFFFFFF] (0xFFFFFFFF = UNMERGEABLE)")
    L = dim.bit_length() - 1
    off = [((1 << (3 * l)) - 1) // 7 for l in range(L + 2)]
    lib = _abi.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    pyr = torch.zeros(off[L + 1], dtype=torch.int32, device=dev)
    pyr[off[L]:] = torch.from_numpy(finest.astype(np.uint32).reshape(-1).view(np.int32)).to(dev)
    _abi.check(lib.lod_merge_pyramid(C.c_void_p(pyr.data_ptr()), L, int(T), current_stream_ptr(dev.index)))
    flat = pyr.cpu().numpy().view(np.uint32).astype(np.int64)
    return [flat[off[l]:off[l + 1]].reshape((1 << l,) * 3) for l in range(L + 1)]


def _linear(cells: np.ndarray, dim: int) -> np.ndarray:
    return (cells[:, 0] * dim + cells[:, 1]) * dim + cells[:, 2]


class Partitioner:
    """The reference Partitioner (partition.py:79-297): composite `run` and its stages.

    `run()` on a fresh partitioner is the fused device build (`lod_split`).  The stage
    methods run the same kernels one stage per call through the staged C ABI
    (`lod_dist_*` with a single rank) and return the reference's intermediate values:
      count()                 -> the finest main counting grid (dim^3 int64)  [K_count]
      extend_overfull_cells() -> {main cell: ExtendedPyramid}                 [extension rounds]
      merge()                 -> main pyramid levels (root first); ep.levels  [merge + node
                                 table + targets + stable distribute: one device program]
      build_targets()         -> the Octree; leaf_nodes / leaf_counts / refs
      insert()                -> checks the leaves (the distribute already ran in merge())
    `bounds` forces the world cube (partition.py:82,87).
    """

    def __init__(self, cloud: PointCloud, config: BuildConfig, bounds: AABB | None = None,
                 device_tree: DeviceTree | None = None):
        if len(cloud) == 0:
            raise ValueError("cannot partition an empty point cloud")
        self.cloud = cloud
        self.config = config
        self.bounds = bounds
        self._dev = device_tree
        self.grid: np.ndarray | None = None
        self.extended: dict[tuple[int, int, int], ExtendedPyramid] = {}
        self.levels: list[np.ndarray] | None = None
        self.refs: list[np.ndarray] | None = None
        self.leaf_nodes: list = []
        self.leaf_counts: list[int] = []
        self.nodes: dict[tuple[int, ...], object] = {}
        self._stage = 0
        self._rb = None
        self._tree = None
        self._cells = None

    # -- composite ---------------------------------------------------------------------

    def run(self) -> Octree:
        if self._stage:   # stages already started: finish them in order
            return self._finish()
        dev = self._dev or DeviceTree()
        cfg = self.config
        d_rec, fmt, n = dev.upload(self.cloud.positions, self.cloud.colors)
        b = None if self.bounds is None else (*self.bounds.min, self.bounds.size)
        dev.split(d_rec, n, fmt, make_config(cfg.T, cfg.initial_depth, cfg.extension_depth, cfg.max_depth), b)
        return GpuOctree(dev, cfg)

    def _finish(self) -> Octree:
        if self._stage < 1:
            self.count()
        if self._stage < 2:
            self.extend_overfull_cells()
        if self._stage < 3:
            self.merge()
        tree = self.build_targets() if self._stage < 4 else self._tree
        if self._stage < 5:
            self.insert()
        return tree

    def _need(self, stage: int, name: str):
        if self._stage != stage:
            raise RuntimeError(f"Partitioner.{name}() called out of order (stages: count, "
                               "extend_overfull_cells, merge, build_targets, insert)")

    # -- stage 1: counting (partition.py:99-105) -----------------------------------------

    def count(self) -> np.ndarray:
        import torch
        from .dist import RankBuilder, _world_cube
        self._need(0, "count")
        cfg = self.config
        dev = self._dev = self._dev or DeviceTree()
        self._d_rec, fmt, n = dev.upload(self.cloud.positions, self.cloud.colors)
        rb = self._rb = RankBuilder(0, 1, dev=dev)
        with torch.cuda.device(dev.device):
            lo, hi = rb.begin(self._d_rec, n, fmt, T=cfg.T, initial_depth=cfg.initial_depth,
                              extension_depth=cfg.extension_depth, max_depth=cfg.max_depth)
            cube = _world_cube(lo, hi) if self.bounds is None else (*self.bounds.min, self.bounds.size)
            span = rb.count(n, cube)
            grid = torch.as_tensor(span, device=f"cuda:{dev.device}").cpu().numpy().view(np.uint32)
        self.bounds = AABB(tuple(float(v) for v in cube[:3]), float(cube[3]))
        dim = 1 << cfg.initial_depth
        self.grid = grid.astype(np.int64).reshape(dim, dim, dim)
        self._stage = 1
        return self.grid

    @property
    def cells(self) -> np.ndarray:
        """(n, 3) finest main-level cell of every point (partition.py:101), from the device keys."""
        if self._cells is None and self._stage >= 1:
            dim = 1 << self.config.initial_depth
            key = self._dev.point_keys(len(self.cloud)).astype(np.int64)
            self._cells = np.stack([key // (dim * dim), (key // dim) % dim, key % dim], axis=1)
        return self._cells

    # -- stage 2: extension rounds (partition.py:109-151) --------------------------------

    def extend_overfull_cells(self) -> dict[tuple[int, int, int], ExtendedPyramid]:
        import torch
        self._need(1, "extend_overfull_cells")
        with torch.cuda.device(self._dev.device):
            while self._rb.extend() is not None:
                pass
        self._stage = 2
        grids = self._dev.ext_grids()
        if not grids:
            return self.extended
        pyr = self._dev.pyramids()
        idx, c16 = self._dev.ext_points()
        o = np.argsort(idx)   # the device lists them in compaction order; the reference's are input order
        idx, c16 = idx[o], c16[o]
        cfg = self.config
        by_anchor = {}
        sorted_by_base = {}
        for g in grids:
            base, ext = int(g.base), int(g.ext)
            anchor = np.array([g.ax, g.ay, g.az], np.int64)
            span = 1 << ext
            lo = int(g.pyr_off) + ((1 << (3 * ext)) - 1) // 7
            finest = pyr[lo:lo + span ** 3].astype(np.int64).reshape(span, span, span)
            if base not in sorted_by_base:   # members: the extension points inside the anchor
                k = _linear(c16 >> (16 - base), 1 << base)
                o = np.argsort(k, kind="stable")
                sorted_by_base[base] = (k[o], o)
            ks, o = sorted_by_base[base]
            key = int(_linear(anchor[None, :], 1 << base)[0])
            a, b = np.searchsorted(ks, [key, key + 1])
            sel = np.sort(o[a:b])
            rel = np.clip((c16[sel] >> (16 - base - ext)) - anchor[None, :] * span, 0, span - 1)
            ep = ExtendedPyramid(cell_path(anchor, base), anchor, ext, finest, idx[sel], rel)
            by_anchor[(base, *anchor.tolist())] = ep
            if base == cfg.initial_depth:
                self.extended[tuple(int(v) for v in anchor)] = ep
        for (base, *anchor), ep in by_anchor.items():   # nest the sub-extensions
            if base == cfg.initial_depth:
                continue
            for (pb, *pa), parent in by_anchor.items():
                if pb + parent.depth == base and all((a >> parent.depth) == p for a, p in zip(anchor, pa)):
                    cell = tuple(int(a - (p << parent.depth)) for a, p in zip(anchor, pa))
                    parent.children[cell] = ep
                    break
        # the reference's dict order (np.argwhere: x-major), which also fixes its leaf numbering
        self.extended = dict(sorted(self.extended.items()))
        for ep in by_anchor.values():
            ep.children = dict(sorted(ep.children.items()))
        return self.extended

    # -- stage 3: merge (partition.py:155-170) -------------------------------------------

    def merge(self) -> list[np.ndarray]:
        import torch
        self._need(2, "merge")
        with torch.cuda.device(self._dev.device):
            self._rb.skeleton()
        self._stage = 3
        pyr = self._dev.pyramids().astype(np.int64)
        L = self.config.initial_depth
        off = lambda l: ((1 << (3 * l)) - 1) // 7
        self.levels = [pyr[off(l):off(l + 1)].reshape((1 << l,) * 3) for l in range(L + 1)]
        grids = {(int(g.base), int(g.ax), int(g.ay), int(g.az)): g for g in self._dev.ext_grids()}
        for ep in self._iter_extended():
            g = grids[(len(ep.anchor_path), *ep.anchor_cell.tolist())]
            ep.levels = [pyr[g.pyr_off + off(l):g.pyr_off + off(l + 1)].reshape((1 << l,) * 3).copy()
                         for l in range(ep.depth + 1)]
            ep.levels[0][0, 0, 0] = UNMERGEABLE   # checked on the device, then cleared there
        return self.levels

    def _iter_extended(self):
        stack = list(self.extended.values())
        while stack:
            ep = stack.pop()
            yield ep
            stack.extend(ep.children.values())

    # -- stage 4: node skeleton + target references (partition.py:174-240) ---------------

    def build_targets(self) -> Octree:
        self._need(3, "build_targets")
        self._tree = GpuOctree(self._dev, self.config)
        self.nodes = {}
        stack = [self._tree.root]
        while stack:
            nd = stack.pop()
            self.nodes[nd.path] = nd
            if nd.children is not None:
                stack.extend(c for c in nd.children if c is not None)
        self.leaf_nodes, self.leaf_counts = [], []
        self.refs = self._refs(self.levels, ())
        for ep in self._iter_extended():
            ep.refs = self._refs(ep.levels, ep.anchor_path)
        self._stage = 4
        return self._tree

    def _refs(self, levels, prefix):
        """Per-level leaf-id grids in the reference's leaf numbering (partition.py:201-231)."""
        refs = []
        for l, grid in enumerate(levels):
            flat = grid.reshape(-1)
            ref = np.full(flat.size, -1, np.int32)
            d = grid.shape[0]
            for lin in np.flatnonzero((flat != 0) & (flat != UNMERGEABLE)):
                path = prefix + cell_path((lin // (d * d), (lin // d) % d, lin % d), l)
                node = self.nodes.get(path)
                if node is None or node.children is not None:
                    raise ConsistencyError(f"leaf cell {path} missing from the device node table")
                ref[lin] = len(self.leaf_nodes)
                self.leaf_nodes.append(node)
                self.leaf_counts.append(int(flat[lin]))
            refs.append(ref)
        return refs

    # -- stage 5: insertion (partition.py:244-287) ---------------------------------------

    def insert(self) -> None:
        """The stable distribute ran with the device merge/targets program; check the result
        like the reference does (partition.py:266-268)."""
        self._need(4, "insert")
        for leaf, c in zip(self.leaf_nodes, self.leaf_counts):
            if len(leaf.point_positions) != c:
                raise ConsistencyError("leaf received a different count than allocated")
        self._stage = 5


def partition(cloud: PointCloud, config: BuildConfig | None = None) -> Octree:
    """Partition a point cloud into an octree with at most T points per leaf (partition.py:300-302)."""
    return Partitioner(cloud, config or BuildConfig()).run()
