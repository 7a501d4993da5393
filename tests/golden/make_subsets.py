"""Subtree-subset goldens for the BASELINE clouds too large for a full CPU run.

Build-container only (runs the REAL, unmodified reference from /root/reference):

    python tests/golden/make_subsets.py [config ...]      # scene500M scene1B cluster2B surface4B

Method (verified 12/12 in the survey's probe 6): for an inner node P of the full tree, the
points inside P's cube, in input order, partitioned by the reference with the full cloud's world
bounds forced -- `Partitioner(subset, BuildConfig(), bounds=world).run()` (partition.py:82,87,
used the same way at test_acceptance.py:229) -- give a tree whose subtree at P is identical to
the full tree's subtree at P, for the split and for every sampling strategy.

Per config:
  1. world bounds over all N points (reference world_bounds_of, model.py:199-209), computed by
     the C restatement of the generators (`oracle/synth.c`, bit-identical to the device
     generator and to `generators.synthetic_rows`, asserted below);
  2. the 256^3 count grid of the full cloud (reference cells_of at initial_depth 8,
     model.py:84-98) -> overfull main cells (extension anchors, partition.py:109-112) and
     counts of every node at depths <= 8;
  3. chosen nodes (depth <= 8, count > T so they are inner in the full tree, pairwise
     disjoint): for cluster2B EVERY extension anchor (the 16 dense clusters and the
     exact-duplicate pile) plus plain sphere nodes; for the others nodes of 1-6M points,
     preferring ones that contain extension anchors;
  4. the subset (rows of the full cloud whose main cell lies in the node, in input order) is run
     through the reference's Partitioner with forced bounds + build_lod for average, random:0
     and first-come; tests/golden/sub_<config>_<path>.json.gz stores per-node digests of the
     subtree at P (same format as make_golden.py), or the reference's exception text.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import multiprocessing as mp
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from oracle.synth import Cloud  # noqa: E402

T = 50_000
MODES = ["average", "random:0", "first-come"]
CHUNK = 1 << 27

# name -> (kind, n, seed); scene1B is the north-star target: the first 1e9 rows of the scene
SUBSET_CONFIGS = {
    "scene500M": ("scene", 500_000_000, 3),
    "scene1B": ("scene", 1_000_000_000, 3),
    "cluster2B": ("cluster", 2_000_000_000, 4),
    "surface4B": ("surface", 4_000_000_000, 5),
}


def _sha(*arrays):
    h = hashlib.sha1()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _ps(path):
    return "".join(str(o) for o in path) or "-"


def cell_path(cell, depth):
    cx, cy, cz = cell
    return tuple(((cx >> b) & 1) | (((cy >> b) & 1) << 1) | (((cz >> b) & 1) << 2) for b in range(depth - 1, -1, -1))


def scan(cloud, n):
    """World bounds (model.py:199-209), the u64 256^3 count grid of the whole cloud and the
    per-axis extents."""
    mn, mx = np.full(3, np.inf), np.full(3, -np.inf)
    for s in range(0, n, CHUNK):
        a, b, bad = cloud.bounds(s, min(CHUNK, n - s))
        assert bad == 0
        mn, mx = np.minimum(mn, a), np.maximum(mx, b)
    ext = float((mx - mn).max())
    world = np.array([mn[0], mn[1], mn[2], ext if ext > 0 else 1.0])
    hist = np.zeros(256 ** 3, np.uint64)
    for s in range(0, n, CHUNK):
        cloud.hist(s, min(CHUNK, n - s), world, 8, hist)
    assert int(hist.sum()) == n
    return world, hist.reshape(256, 256, 256), mx - mn


def level_counts(h8, d):
    k = 1 << (8 - d)
    return h8.reshape(1 << d, k, 1 << d, k, 1 << d, k).sum(axis=(1, 3, 5))


def choose(name, h8, ext_hi=None):
    """[(depth, (cx, cy, cz), count)] of disjoint inner nodes (see module docstring)."""
    anchors = np.argwhere(h8 > T)
    chosen = []

    def overlaps(d, c):
        for d2, c2, _ in chosen:
            m = min(d, d2)
            if all((c[a] >> (d - m)) == (c2[a] >> (d2 - m)) for a in range(3)):
                return True
        return False

    def anchors_in(d, c):
        k = 8 - d
        return int(np.all((anchors >> k) == np.asarray(c), axis=1).sum()) if len(anchors) else 0

    if name == "cluster2B":
        for c in anchors:
            chosen.append((8, tuple(int(v) for v in c), int(h8[tuple(c)])))
        lc = level_counts(h8, 4)
        for c in np.argwhere((lc > 1_000_000) & (lc < 3_000_000)):
            c = tuple(int(v) for v in c)
            if not overlaps(4, c) and anchors_in(4, c) == 0:
                chosen.append((4, c, int(lc[c])))
            if sum(1 for d, _, _ in chosen if d == 4) == 2:
                break
        return chosen
    lo, hi = 1_000_000, 6_000_000
    cands = []
    for d in range(2, 8):
        lc = level_counts(h8, d)
        for c in np.argwhere((lc > lo) & (lc < hi)):
            c = tuple(int(v) for v in c)
            cands.append((anchors_in(d, c), d, c, int(lc[c])))
    # most extension anchors first, then one anchor-free node, then the deepest remaining
    cands.sort(key=lambda x: (-x[0], x[1], x[2]))
    for na, d, c, cnt in cands:
        if not overlaps(d, c):
            chosen.append((d, c, cnt))
            break
    for na, d, c, cnt in cands:
        if na == 0 and not overlaps(d, c):
            chosen.append((d, c, cnt))
            break
    for na, d, c, cnt in sorted(cands, key=lambda x: (-x[1], -x[3])):
        if not overlaps(d, c):
            chosen.append((d, c, cnt))
            break
    # a node on the world's max face along the extent-defining axis (clipped max-face points)
    axis = int(np.argmax([ext_hi[a] for a in range(3)])) if ext_hi is not None else 0
    for d in range(7, 1, -1):
        lc = level_counts(h8, d)
        face = [(int(lc[c]), c) for c in map(tuple, np.argwhere(lc > T)) if c[axis] == (1 << d) - 1]
        face = [(k, tuple(int(v) for v in c)) for k, c in face if k < hi and not overlaps(d, tuple(int(v) for v in c))]
        if face:
            k, c = max(face)
            chosen.append((d, c, k))
            break
    return chosen


def extract(cloud, n, world, chosen, outdir):
    """Rows of each chosen node in input order -> <outdir>/<i>_pos.npy / _col.npy / _idx.npy."""
    lut = np.full(256 ** 3, -1, np.int16)
    lut3 = lut.reshape(256, 256, 256)
    for i, (d, c, _) in enumerate(chosen):
        k = 8 - d
        lut3[c[0] << k:(c[0] + 1) << k, c[1] << k:(c[1] + 1) << k, c[2] << k:(c[2] + 1) << k] = i
    parts = [[] for _ in chosen]
    for s in range(0, n, CHUNK):
        sel = cloud.select(s, min(CHUNK, n - s), world, 8, lut)
        hit = np.flatnonzero(sel >= 0)
        ids = sel[hit]
        order = np.argsort(ids, kind="stable")
        hit, ids = hit[order], ids[order]
        bounds = np.searchsorted(ids, np.arange(len(chosen) + 1))
        for i in range(len(chosen)):
            parts[i].append(hit[bounds[i]:bounds[i + 1]].astype(np.uint64) + np.uint64(s))
    files = []
    for i, (d, c, cnt) in enumerate(chosen):
        idx = np.concatenate(parts[i])
        assert len(idx) == cnt, (i, len(idx), cnt)
        pos, col = cloud.rows_idx(idx)
        base = os.path.join(outdir, f"{i}")
        np.save(base + "_pos.npy", pos)
        np.save(base + "_col.npy", col)
        files.append((base, _sha(idx)))
    return files


def _offender(tree, strat):
    """Path of the node build_lod raised on: the first inner node in its order (deepest first,
    DFS preorder inside a depth; sampling.py:171) whose children's samples reach 2^20."""
    if strat != "random":
        return None
    for nd in sorted(tree.inner_nodes(), key=lambda n: n.depth, reverse=True):
        s_ = sum(c.sample_count for _, c in nd.existing_children())
        if s_ >= 1 << 20:
            return _ps(nd.path)
    return None


def skeleton(name, world, h8, max_depth=4):
    """Nodes of the FULL tree at depths <= max_depth, from the reference's own merge rule:
    lodforge.partition.merge_pyramid on the full 256^3 count grid with every overfull cell
    flagged UNMERGEABLE (partition.py:155-161; an extended anchor is always inner), node =
    non-zero pyramid cell (partition.py:201-231), bounds = lodforge.model.bounds_at.
    path -> [kind, points in the node's cube, bounds hex]."""
    from lodforge.model import AABB, bounds_at
    from lodforge.partition import UNMERGEABLE, merge_pyramid
    finest = h8.astype(np.int64)
    finest[finest > T] = UNMERGEABLE
    levels = merge_pyramid(finest, T)
    wb = AABB((float(world[0]), float(world[1]), float(world[2])), float(world[3]))
    out = {}
    for d in range(0, max_depth + 1):
        lc = level_counts(h8, d) if d < 8 else h8
        for c in np.argwhere(levels[d] != 0):
            c = tuple(int(v) for v in c)
            path = cell_path(c, d)
            b = bounds_at(wb, path)
            kind = "I" if int(levels[d][c]) == UNMERGEABLE else "L"
            out[_ps(path)] = [kind, int(lc[c]), [float(v).hex() for v in b.min] + [float(b.size).hex()]]
    return out


def run_subset(job):
    """Reference Partitioner(subset, BuildConfig(), bounds=world) + build_lod (one process)."""
    from lodforge.errors import ConsistencyError
    from lodforge.ingest import PointCloud
    from lodforge.model import AABB, BuildConfig
    from lodforge.partition import Partitioner
    from lodforge.sampling import build_lod

    name, world, depth, cell, base, idx_sha, n_full = job
    t0 = time.time()
    pos = np.load(base + "_pos.npy")
    col = np.load(base + "_col.npy")
    cloud = PointCloud(pos.astype(np.float64), col)
    bounds = AABB((float(world[0]), float(world[1]), float(world[2])), float(world[3]))
    tree = Partitioner(cloud, BuildConfig(), bounds=bounds).run()
    prefix = cell_path(cell, depth)
    pstr = _ps(prefix)

    def inside(nd):
        return tuple(nd.path[:depth]) == prefix

    split = {}
    for nd in tree.iter_nodes():
        if not inside(nd):
            continue
        b = [float(v).hex() for v in nd.bounds.min] + [float(nd.bounds.size).hex()]
        if nd.is_leaf:
            split[_ps(nd.path)] = ["L", nd.point_count, bool(nd.oversized), b,
                                   _sha(nd.point_positions, nd.point_colors)]
        else:
            split[_ps(nd.path)] = ["I", 0, False, b, ""]
    modes = {}
    for mode in MODES:
        strat, _, seed = mode.partition(":")
        try:
            build_lod(tree, strat, int(seed or 0))
            modes[mode] = {_ps(nd.path): [nd.voxel_count, _sha(nd.voxel_coords, nd.voxel_colors)]
                           for nd in tree.inner_nodes() if inside(nd)}
        except ConsistencyError as e:
            modes[mode] = {"error": str(e), "at": _offender(tree, strat)}
    out = {"config": name, "n_full": n_full, "world": [float(v).hex() for v in world], "depth": depth,
           "cell": list(cell), "path": pstr, "n": len(pos), "index_sha": idx_sha,
           "input_sha": _sha(cloud.positions, cloud.colors), "T": T, "split": split, "modes": modes,
           "seconds": round(time.time() - t0, 1)}
    fn = os.path.join(HERE, f"sub_{name}_{pstr}.json.gz")
    with gzip.open(fn, "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    for suf in ("_pos.npy", "_col.npy"):
        os.remove(base + suf)
    return name, pstr, len(pos), len(split), out["seconds"], {m: ("error" in v) for m, v in modes.items()}


def main(argv):
    names = [a for a in argv if not a.startswith("--")] or list(SUBSET_CONFIGS)
    from paper_2302_14801_b200.generators import synthetic_rows
    tmp = tempfile.mkdtemp(prefix="subsets_", dir="/tmp")
    jobs = []
    for name in names:
        kind, n, seed = SUBSET_CONFIGS[name]
        cloud = Cloud(kind, seed)
        for s in (0, n - 4096):   # the C generator is the numpy one, bit for bit
            p, c = cloud.rows(s, 4096)
            p2, c2 = synthetic_rows(kind, seed, s, 4096)
            assert np.array_equal(p.view(np.uint32), p2.view(np.uint32)) and np.array_equal(c, c2)
        t0 = time.time()
        world, h8, extents = scan(cloud, n)
        chosen = choose(name, h8, ext_hi=extents)
        full = {"config": name, "kind": kind, "n": n, "seed": seed, "T": T,
                "world": [float(v).hex() for v in world], "extents": [float(v).hex() for v in extents],
                "anchors": int((h8 > T).sum()), "skeleton_depth": 4, "skeleton": skeleton(name, world, h8),
                "subsets": [_ps(cell_path(c, d)) for d, c, _ in chosen]}
        with gzip.open(os.path.join(HERE, f"full_{name}.json.gz"), "wt") as f:
            json.dump(full, f, separators=(",", ":"))
        print(f"{name}: world {world.tolist()} scan {time.time() - t0:.0f}s; "
              f"{int((h8 > T).sum())} anchors; chosen {[(d, c, k) for d, c, k in chosen]}", flush=True)
        outdir = os.path.join(tmp, name)
        os.makedirs(outdir)
        files = extract(cloud, n, world, chosen, outdir)
        for (d, c, cnt), (base, isha) in zip(chosen, files):
            jobs.append((name, world.tolist(), d, c, base, isha, n))
        print(f"{name}: extracted {sum(k for _, _, k in chosen)} points in {time.time() - t0:.0f}s", flush=True)
    jobs.sort(key=lambda j: -os.path.getsize(j[4] + "_pos.npy"))
    with mp.get_context("fork").Pool(min(8, os.cpu_count() or 1), maxtasksperchild=1) as pool:
        for r in pool.imap_unordered(run_subset, jobs):
            print(r, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
