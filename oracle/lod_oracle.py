"""CPU ORACLE -- test infrastructure only.

A numpy restatement of the reference's LOD-construction path (the `lodforge`
package: `pkg/src/lodforge/partition.py` + `sampling.py` + the fp64 geometry in
`model.py`), used to check the CUDA path.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
leg may import it; the product path (`paper_2302_14801_b200`) never does.

Parity is pinned: `tests/test_oracle_golden.py` checks this module against
digests produced by running the real reference (`tests/golden/make_golden.py`)
on the reference's own test datasets and on the BASELINE configs.

Layout of a split result (`Split`):
  nodes: dict path(tuple) -> Node(kind 'leaf'|'inner', count, oversized, idx)
  where idx = input indices of a leaf's points in input order (partition.py:262
  uses a stable argsort, so leaves keep input order).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

UNMERGEABLE = 0xFFFFFFFF      # partition.py:20
GRID = 128                    # model.py:18
RANDOM_LIMIT = 1 << 20        # sampling.py:18

_GOLDEN = 0x9E3779B97F4A7C15
_MASK = (1 << 64) - 1


class ConsistencyError(Exception):
    """Mirror of lodforge.errors.ConsistencyError (errors.py:5-6)."""


# ---------------------------------------------------------------------------
# geometry (model.py)
# ---------------------------------------------------------------------------


def world_bounds(pos: np.ndarray):
    """(min xyz, size) cube around the points -- model.py:199-209."""
    pos = np.asarray(pos, np.float64)
    if pos.size == 0:
        raise ValueError("cannot bound an empty point set")
    if not np.isfinite(pos).all():
        raise ValueError("point coordinates must be finite")
    lo = pos.min(axis=0)
    ext = float((pos.max(axis=0) - lo).max())
    return (float(lo[0]), float(lo[1]), float(lo[2])), (ext if ext > 0 else 1.0)


def grid_cells(pos, lo, size, dim, check=True):
    """clip(floor((p - lo) / size * dim), 0, dim - 1) -- model.py:84-98, partition.py:134-135."""
    rel = np.asarray(pos, np.float64) - np.asarray(lo, np.float64)
    if check and ((rel < 0).any() or (rel > size).any()):
        raise ConsistencyError("point outside bounds during grid projection")
    c = np.floor(rel / size * dim)
    return np.clip(c, 0, dim - 1).astype(np.int64)


def node_bounds(lo, size, path):
    """Sequential child_bounds fold (model.py:62-81); not the closed form (hazard H2)."""
    x, y, z = lo
    s = size
    for o in path:
        h = s / 2
        x, y, z = x + h * (o & 1), y + h * ((o >> 1) & 1), z + h * ((o >> 2) & 1)
        s = h
    return (x, y, z), s


def _lin(c, dim):
    return (c[:, 0] * dim + c[:, 1]) * dim + c[:, 2]          # partition.py:23-24


def _digits(cell, level):
    """Octant digits of an integer cell at `level`, msb first -- partition.py:27-33."""
    cx, cy, cz = (int(v) for v in cell)
    return tuple(((cx >> s) & 1) | (((cy >> s) & 1) << 1) | (((cz >> s) & 1) << 2)
                 for s in range(level - 1, -1, -1))


# ---------------------------------------------------------------------------
# split (partition.py)
# ---------------------------------------------------------------------------


def merge_levels(finest: np.ndarray, T: int) -> list[np.ndarray]:
    """Bottom-up 2x2x2 merge with the UNMERGEABLE sentinel, root level first -- partition.py:36-61.

    Group rule: no flagged child and 0 < sum < T -> parent = sum, children := 0;
    any flagged child or sum > 0 -> parent = UNMERGEABLE; else parent = 0.
    """
    cur = np.array(finest, dtype=np.int64)
    out = [cur]
    while cur.shape[0] > 1:
        h = cur.shape[0] // 2
        flag = cur == UNMERGEABLE
        blocks = np.where(flag, 0, cur).reshape(h, 2, h, 2, h, 2)
        s = blocks.sum(axis=(1, 3, 5))
        anyflag = flag.reshape(h, 2, h, 2, h, 2).any(axis=(1, 3, 5))
        merged = (~anyflag) & (s > 0) & (s < T)
        parent = np.where(merged, s, np.where(anyflag | (s > 0), UNMERGEABLE, 0))
        clear = np.broadcast_to(merged[:, None, :, None, :, None], (h, 2, h, 2, h, 2))
        cur[clear.reshape(2 * h, 2 * h, 2 * h)] = 0
        cur = parent
        out.append(cur)
    return out[::-1]


@dataclass
class Node:
    kind: str                      # "leaf" | "inner"
    count: int = 0                 # leaf point count
    oversized: bool = False
    idx: np.ndarray | None = None  # leaf: input indices, input order


@dataclass
class _Tier:
    """One counting pyramid: the main grid or an extension of an overfull cell (partition.py:64-76)."""

    prefix: tuple                  # path of the tier's root cell
    levels_n: int                  # number of levels below the root (finest grid = 2^levels_n)
    idx: np.ndarray                # member points, input order
    fine: np.ndarray               # (n, 3) finest-level cells relative to the tier root
    counts: np.ndarray = None
    subs: dict = field(default_factory=dict)   # finest cell -> child _Tier
    levels: list = None


@dataclass
class Split:
    world: tuple                   # (lo xyz, size)
    config: dict
    nodes: dict                    # path -> Node
    top: object = None             # the main _Tier (stage values: counts, subs, levels, refs)


def split(pos, T=50_000, initial_depth=8, extension_depth=4, max_depth=16, bounds=None) -> Split:
    """Hierarchical counting-sort split -- Partitioner.run (partition.py:291-297)."""
    pos = np.asarray(pos, np.float64)
    n = len(pos)
    if n == 0:
        raise ValueError("cannot partition an empty point cloud")       # partition.py:83-84
    lo, size = bounds if bounds is not None else world_bounds(pos)
    dim = 1 << initial_depth
    top_cells = grid_cells(pos, lo, size, dim)                          # count(), partition.py:99-105
    top = _Tier((), initial_depth, np.arange(n), top_cells)
    top.counts = np.bincount(_lin(top_cells, dim), minlength=dim ** 3).reshape(dim, dim, dim)

    def extend(tier: _Tier, depth_at_fine: int):
        """Grow a 2^ext sub-grid under every overfull finest cell -- partition.py:109-151."""
        if depth_at_fine >= max_depth:
            return
        span_fine = 1 << tier.levels_n
        keys = _lin(tier.fine, span_fine)
        for cell in np.argwhere(tier.counts > T):
            k = (cell[0] * span_fine + cell[1]) * span_fine + cell[2]
            members = tier.idx[keys == k]                                # input order kept
            ext = min(extension_depth, max_depth - depth_at_fine)
            full = grid_cells(pos[members], lo, size, 1 << (depth_at_fine + ext), check=False)
            anchor = _abs_cell(tier, cell)
            rel = np.clip(full - anchor[None, :] * (1 << ext), 0, (1 << ext) - 1)
            sub = _Tier(tier.prefix + _digits(cell, tier.levels_n), ext, members, rel)
            sp = 1 << ext
            sub.counts = np.bincount(_lin(rel, sp), minlength=sp ** 3).reshape(sp, sp, sp)
            sub.anchor = anchor
            tier.subs[tuple(int(v) for v in cell)] = sub
            extend(sub, depth_at_fine + ext)

    def _abs_cell(tier, cell):
        base = getattr(tier, "anchor", np.zeros(3, np.int64))
        return base * (1 << tier.levels_n) + np.asarray(cell, np.int64)

    top.anchor = np.zeros(3, np.int64)
    if max_depth > initial_depth:
        extend(top, initial_depth)

    def merge(tier: _Tier):                                              # partition.py:155-170
        fin = tier.counts.astype(np.int64).copy()
        for cell, sub in tier.subs.items():
            merge(sub)
            fin[cell] = UNMERGEABLE
        tier.levels = merge_levels(fin, T)
        if tier.prefix and int(tier.levels[0].flat[0]) != UNMERGEABLE:
            raise ConsistencyError("extended pyramid root must be unmergeable")

    merge(top)

    nodes: dict = {}
    leaf_of = np.full(n, -1, np.int64)
    leaf_paths: list = []

    def materialize(tier: _Tier):                                        # partition.py:201-231
        depth_fine = len(tier.prefix) + tier.levels_n
        tier.refs = []
        for l, grid in enumerate(tier.levels):
            d = grid.shape[0]
            flat = grid.reshape(-1)
            ref = np.full(flat.size, -1, np.int64)
            for lin in np.flatnonzero(flat):
                v = int(flat[lin])
                path = tier.prefix + _digits((lin // (d * d), (lin // d) % d, lin % d), l)
                if path in nodes:   # tier root duplicates the anchor's inner node
                    continue
                if v == UNMERGEABLE:
                    nodes[path] = Node("inner")
                else:
                    over = v > T
                    if over and not (depth_fine >= max_depth and l == len(tier.levels) - 1):
                        raise ConsistencyError("oversized leaf away from max depth")
                    nodes[path] = Node("leaf", v, over)
                    ref[lin] = len(leaf_paths)
                    leaf_paths.append(path)
            tier.refs.append(ref)
        for sub in tier.subs.values():
            materialize(sub)

    materialize(top)
    if () not in nodes:
        raise ConsistencyError("partition produced no root node")
    for path in nodes:                                                   # partition.py:233-240
        if path and (path[:-1] not in nodes or nodes[path[:-1]].kind != "inner"):
            raise ConsistencyError(f"node {path} has no inner parent")

    def resolve(tier: _Tier):
        """Walk each member up its tier's pyramid to the first leaf cell -- partition.py:244-287."""
        for sub in tier.subs.values():
            resolve(sub)
        local = leaf_of[tier.idx]
        for l in range(tier.levels_n, -1, -1):
            todo = np.flatnonzero(local < 0)
            if todo.size == 0:
                break
            c = tier.fine[todo] >> (tier.levels_n - l)
            local[todo] = tier.refs[l][_lin(c, 1 << l)]
        if (local < 0).any():
            raise ConsistencyError("point did not resolve to a leaf node")
        leaf_of[tier.idx] = local

    resolve(top)
    order = np.argsort(leaf_of, kind="stable")
    bounds_ = np.searchsorted(leaf_of[order], np.arange(len(leaf_paths) + 1))
    for i, path in enumerate(leaf_paths):
        sel = order[bounds_[i]:bounds_[i + 1]]
        if len(sel) != nodes[path].count:
            raise ConsistencyError("leaf received a different count than allocated")
        nodes[path].idx = sel
    cfg = dict(T=T, initial_depth=initial_depth, extension_depth=extension_depth, max_depth=max_depth)
    return Split(((float(lo[0]), float(lo[1]), float(lo[2])), float(size)), cfg, nodes, top)


# ---------------------------------------------------------------------------
# voxel sampling (sampling.py)
# ---------------------------------------------------------------------------


def mix64_array(x):
    z = np.asarray(x, np.uint64) + np.uint64(_GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def path_hash(seed, path):
    """rng.py:48-53."""
    def mix(x):
        z = (x + _GOLDEN) & _MASK
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    key = seed & _MASK
    for o in path:
        key = mix((key * 8 + o + 1) & _MASK)
    return key


def child_gpos(sp: Split, pos, col, vox, path):
    """Canonical sample list of an inner node -- project_child_samples, sampling.py:21-47.

    Returns (gpos (S,3) float64 grid positions in [0, 128), colors (S,3) uint8), children in
    octant order, each child's samples in stored order (the sample ordinals, sampling.py:5-6).
    """
    lo, size = node_bounds(sp.world[0], sp.world[1], path)
    lo = np.asarray(lo)
    gp, cols = [], []
    for o in range(8):
        cp = path + (o,)
        ch = sp.nodes.get(cp)
        if ch is None:
            continue
        if ch.kind == "leaf":
            if ch.count == 0:
                raise ConsistencyError(f"child {cp} has no samples")          # sampling.py:34-35
            g = (pos[ch.idx] - lo) / size * float(GRID)                        # sampling.py:37
            gp.append(np.clip(g, 0.0, np.nextafter(float(GRID), 0.0)))         # sampling.py:30,38
            cols.append(col[ch.idx])
        else:
            vc, vcol = vox[cp]
            if len(vc) == 0:
                raise ConsistencyError(f"child {cp} has no samples")
            off = np.array([64.0 * (o & 1), 64.0 * ((o >> 1) & 1), 64.0 * ((o >> 2) & 1)])
            gp.append(off + (vc.astype(np.float64) + 0.5) / 2.0)             # sampling.py:41-44
            cols.append(vcol)
    return np.concatenate(gp), np.concatenate(cols)


def child_samples(sp: Split, pos, col, vox, path):
    """(cells (S,3) int64 in the node's 128^3 grid, colors) -- sampling.py:50-52 on child_gpos."""
    gp, cols = child_gpos(sp, pos, col, vox, path)
    return np.floor(gp).astype(np.int64), cols


def _keys(cells):
    return (cells[:, 0] * GRID + cells[:, 1]) * GRID + cells[:, 2]


def _coords(keys):
    return np.stack([keys // (GRID * GRID), (keys // GRID) % GRID, keys % GRID], 1).astype(np.uint8)


def extract_random(cells, cols, seed, node_hash):
    """Max (rand12 | ordinal20) per cell, voxels by ascending key -- sampling.py:69-85."""
    s = len(cells)
    if s >= RANDOM_LIMIT:
        raise ConsistencyError(f"{s} samples exceed the 20-bit index limit of random sampling")
    keys = _keys(cells)
    ords = np.arange(s, dtype=np.uint64)
    r32 = (mix64_array(np.uint64((seed ^ node_hash) & _MASK) ^ ords) >> np.uint64(32)).astype(np.uint32)
    enc = (r32 & np.uint32(0xFFF00000)) | (ords.astype(np.uint32) & np.uint32(0xFFFFF))
    order = np.lexsort((enc, keys))
    sk = keys[order]
    last = np.r_[sk[1:] != sk[:-1], True]
    return _coords(sk[last]), cols[order[last]].copy()


def extract_average(cells, cols):
    """Exact integer channel sums per cell, (2*sum + n) // (2*n) -- sampling.py:88-97."""
    keys = _keys(cells)
    uk, inv = np.unique(keys, return_inverse=True)
    cnt = np.bincount(inv).astype(np.int64)
    out = np.empty((len(uk), 3), np.uint8)
    for ch in range(3):
        sums = np.bincount(inv, weights=cols[:, ch].astype(np.float64)).astype(np.int64)
        out[:, ch] = (2 * sums + cnt) // (2 * cnt)
    return _coords(uk), out


def extract_first_come(cells, cols):
    """Smallest ordinal per cell wins; voxels listed by winning ordinal -- sampling.py:61-66."""
    _, first = np.unique(_keys(cells), return_index=True)
    win = np.sort(first)
    return cells[win].astype(np.uint8), cols[win].copy()


def extract_weighted(gpos, cols):
    """Distance-weighted 2x2x2 mean over occupied cells -- sampling.py:100-133.

    Same numpy operations in the same order as the reference, so the fp64 sums agree
    bit-for-bit here (the GPU path is held to +-1 per channel, SPEC.md)."""
    g = GRID
    base = np.clip(np.floor(gpos - 0.5), 0, g - 2).astype(np.int64)
    kp, wp, wcp = [], [], []
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                cell = base + np.array([dx, dy, dz])
                d = np.sqrt(((gpos - (cell + 0.5)) ** 2).sum(axis=1))
                w = np.clip(1.0 - d, 0.0, 1.0)
                kp.append((cell[:, 0] * g + cell[:, 1]) * g + cell[:, 2])
                wp.append(w)
                wcp.append(w[:, None] * cols)
    keys = np.concatenate(kp)
    weights = np.concatenate(wp)
    wcols = np.concatenate(wcp)
    uk, inv = np.unique(keys, return_inverse=True)
    wsum = np.bincount(inv, weights=weights)
    csum = np.stack([np.bincount(inv, weights=wcols[:, ch]) for ch in range(3)], axis=1)
    occupied = np.unique(_keys(np.floor(gpos).astype(np.int64)))
    at = np.searchsorted(uk, occupied)
    denom = wsum[at]
    if (denom <= 0).any():
        raise ConsistencyError("occupied cell accumulated zero weight")          # sampling.py:129-130
    mean = np.floor(csum[at] / denom[:, None] + 0.5)
    return _coords(occupied), np.clip(mean, 0, 255).astype(np.uint8)


MODES = ("first-come", "random", "average", "weighted")   # model.py:127 STRATEGIES


def voxelize(sp: Split, pos, col, mode="average", seed=0):
    """Fill inner nodes deepest first -- build_lod, sampling.py:165-176.

    Returns dict path -> (coords (m,3) u8, colors (m,3) u8) in stored order.
    """
    mode = {"color_filter": "average"}.get(mode, mode)
    if mode not in MODES:
        raise ValueError(f"unknown sampling strategy: {mode}")
    pos = np.asarray(pos, np.float64)
    col = np.asarray(col, np.uint8)
    vox: dict = {}
    inner = sorted((p for p, nd in sp.nodes.items() if nd.kind == "inner"), key=len, reverse=True)
    for path in inner:
        gp, cols = child_gpos(sp, pos, col, vox, path)
        cells = np.floor(gp).astype(np.int64)
        if mode == "random":
            vox[path] = extract_random(cells, cols, seed, path_hash(seed, path))
        elif mode == "average":
            vox[path] = extract_average(cells, cols)
        elif mode == "first-come":
            vox[path] = extract_first_come(cells, cols)
        else:
            vox[path] = extract_weighted(gp, cols)
    return vox


# ---------------------------------------------------------------------------
# canonical digests (shared with the golden fixtures and the GPU tests)
# ---------------------------------------------------------------------------


def _sha(*arrays) -> str:
    h = hashlib.sha1()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def path_str(path) -> str:
    return "".join(str(o) for o in path) or "-"


def split_digest(sp: Split, pos, col) -> dict:
    """path -> [kind, count, oversized, bounds-hex, sha1(leaf positions f64 || colors u8)]."""
    pos = np.asarray(pos, np.float64)
    col = np.asarray(col, np.uint8)
    out = {}
    for path, nd in sp.nodes.items():
        lo, s = node_bounds(sp.world[0], sp.world[1], path)
        b = [float(v).hex() for v in lo] + [float(s).hex()]
        if nd.kind == "leaf":
            out[path_str(path)] = ["L", nd.count, bool(nd.oversized), b, _sha(pos[nd.idx], col[nd.idx])]
        else:
            out[path_str(path)] = ["I", 0, False, b, ""]
    return out


def voxel_digest(vox: dict) -> dict:
    """path -> [m, sha1(coords || colors)]."""
    return {path_str(p): [len(c), _sha(c, k)] for p, (c, k) in vox.items()}
