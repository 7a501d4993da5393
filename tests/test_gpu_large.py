"""GPU parity at the BASELINE's large configs (scene500M, scene@1B = the north-star target,
cluster2B, surface4B), where a full CPU run of the reference does not fit the host.

Evidence, all from the REAL reference (tests/golden/make_subsets.py):
  * sub_<config>_<path>.json.gz -- subtree-subset goldens: the reference's
    Partitioner(subset, BuildConfig(), bounds=world) (partition.py:82,87) + build_lod on the
    points inside an inner node, which reproduces the full tree's subtree at that node.  For
    cluster2B EVERY extension anchor (16 dense clusters + the duplicate pile) is one.
  * full_<config>.json.gz -- the full cloud's world bounds and its skeleton at depths <= 4
    from the reference's own merge_pyramid on the exact 256^3 count grid + bounds_at.

Tests:
  1. test_full_cloud: the WHOLE cloud generated in HBM, split + voxelized on one B200 through
     the C ABI, then every golden subtree compared node by node (fp64 bounds, counts, oversized
     flags, leaf points in input order, voxels in stored order for average / random / first-come)
     plus the depth <= 4 skeleton, plus an inductive check of the shallow inner nodes (each one
     re-sampled by the oracle from its children's GPU outputs).  surface4B's working set
     (~56 B/pt = 224 GB) does not fit one GPU: its full build is the multi-GPU config.
  2. test_subsets_forced_bounds: each subset extracted on the device from the generated cloud
     (its row indices hashed against the golden), then driven through the public drop-in
     `Partitioner(cloud, BuildConfig(), bounds=AABB)` + `build_lod`, compared with the golden.
"""
import gc
import glob
import gzip
import json
import os

import numpy as np
import pytest

from helpers import (cell_path_str, decode_voxels, device_subtree_split, device_subtree_voxels, diff_dicts, sha,
                     subtree_index, tree_split_digest, tree_voxel_digest)

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODES = ["average", "random:0", "first-come"]
RANDOM_LIMIT = 1 << 20


def _load(fn):
    with gzip.open(fn, "rt") as f:
        return json.load(f)


FULL = sorted(os.path.basename(f)[5:-8] for f in glob.glob(os.path.join(GOLDEN, "full_*.json.gz")))


def _subs(name):
    return [_load(f) for f in sorted(glob.glob(os.path.join(GOLDEN, f"sub_{name}_*.json.gz")))]


def _world(full):
    return [float.fromhex(v) for v in full["world"]]


def _free_bytes():
    import torch
    free, _ = torch.cuda.mem_get_info()
    return free


def _mode(mode):
    from paper_2302_14801_b200.sampling import _mode_code
    strat, _, seed = mode.partition(":")
    return strat, _mode_code(strat), int(seed or 0)


def _expected_offender(nodes):
    """Reference build_lod order (deepest first, DFS preorder = path order inside a depth,
    sampling.py:171) -> (S, path) of the first inner node whose children's samples reach
    2^20 (sampling.py:73-75), from a completed tree's node table (samples = leaf points or
    child voxels; occupancy is the same for every strategy)."""
    inner = [k for k in range(len(nodes)) if not nodes[k]["flags"] & 1]
    paths = {k: cell_path_str(nodes[k]["cell"], int(nodes[k]["depth"])) for k in inner}
    inner.sort(key=lambda k: (-int(nodes[k]["depth"]), paths[k]))
    for k in inner:
        s = sum(int(nodes[c]["count"]) for c in nodes[k]["child"] if c >= 0)
        if s >= RANDOM_LIMIT:
            return s, paths[k]
    return None


def _oracle_node(dev, nodes, k, strat, seed):
    """The reference's sampling of inner node k (sampling.py:21-133, via the oracle's extract
    functions) applied to its children's GPU outputs."""
    from oracle import lod_oracle as O
    from paper_2302_14801_b200.device import unpack_records
    fmt = dev.info().point_format
    nd = nodes[k]
    lo, size = np.asarray(nd["min"], np.float64), float(nd["size"])
    gp, cols = [], []
    for o in range(8):
        c = int(nd["child"][o])
        if c < 0:
            continue
        ch = nodes[c]
        if ch["flags"] & 1:
            pos, col = unpack_records(dev.leaf_range(int(ch["first"]), int(ch["count"])), fmt)
            g = (pos - lo) / size * 128.0
            gp.append(np.clip(g, 0.0, np.nextafter(128.0, 0.0)))
        else:
            vc, col = decode_voxels(dev.voxel_range(int(ch["first"]), int(ch["count"])))
            off = np.array([64.0 * (o & 1), 64.0 * ((o >> 1) & 1), 64.0 * ((o >> 2) & 1)])
            gp.append(off + (vc.astype(np.float64) + 0.5) / 2.0)
        cols.append(col)
    gp, cols = np.concatenate(gp), np.concatenate(cols)
    cells = np.floor(gp).astype(np.int64)
    path = tuple(int(ch) for ch in cell_path_str(nd["cell"], int(nd["depth"])).replace("-", ""))
    if strat == "random":
        return O.extract_random(cells, cols, seed, O.path_hash(seed, path))
    if strat == "average":
        return O.extract_average(cells, cols)
    return O.extract_first_come(cells, cols)


def _structure_properties(nodes, n, T, max_depth):
    """Acceptance criteria 01/02 (test_acceptance.py:71-95) on the full node table:
    conservation, capacity (oversized only at max depth), merging maximality, and every inner
    node linked to its existing children."""
    leaf = (nodes["flags"] & 1) == 1
    over = (nodes["flags"] & 2) == 2
    cnt = nodes["count"].astype(np.int64)
    assert int(cnt[leaf].sum()) == n, "conservation"
    assert (cnt[leaf & ~over] <= T).all(), "capacity"
    assert (nodes["depth"][over] == max_depth).all(), "oversized leaf away from max depth"
    ch = nodes["child"]
    inner = np.flatnonzero(~leaf)
    kids = ch[inner]
    assert ((kids >= 0).any(axis=1)).all(), "inner node without children"
    all_leaf = np.array([all(leaf[c] for c in row if c >= 0) for row in kids])
    sums = np.array([int(cnt[[c for c in row if c >= 0]].sum()) for row in kids])
    assert (sums[all_leaf] >= T).all(), "merging maximality"


def _occupancy_sums(dev, nodes):
    """Per inner node: (voxel count, sum of keys, sum of squared keys mod 2^64) -- order-
    independent, so first-come's ordinal order compares with the others' key order
    (criterion 05, test_acceptance.py:154-166)."""
    inner = np.flatnonzero((nodes["flags"] & 1) == 0)
    keys = dev.voxels()[:, 0].astype(np.uint64)
    with np.errstate(over="ignore"):
        c1 = np.concatenate([np.zeros(1, np.uint64), np.cumsum(keys, dtype=np.uint64)])
        c2 = np.concatenate([np.zeros(1, np.uint64), np.cumsum(keys * keys, dtype=np.uint64)])
        f = nodes["first"][inner].astype(np.int64)
        e = f + nodes["count"][inner].astype(np.int64)
        s1, s2 = c1[e] - c1[f], c2[e] - c2[f]
    return {int(i): (int(e[j] - f[j]), int(s1[j]), int(s2[j])) for j, i in enumerate(inner)}


@pytest.mark.parametrize("name", FULL)
def test_full_cloud(name):
    import torch
    from paper_2302_14801_b200 import ConsistencyError
    from paper_2302_14801_b200._abi import LOD_POINTS_F32
    from paper_2302_14801_b200.device import DeviceTree, generate_device, make_config

    full = _load(os.path.join(GOLDEN, f"full_{name}.json.gz"))
    n = full["n"]
    gc.collect()
    torch.cuda.empty_cache()
    free = _free_bytes()
    if n * 88 > free:   # input 16 B/pt + the tree's buffers (~70 B/pt at cluster2B)
        pytest.skip(f"{name}: the single-GPU working set (~88 B/pt = {n * 88 / 1e9:.0f} GB) exceeds the "
                    f"{free / 1e9:.0f} GB free on this B200; its full build is the multi-GPU config "
                    "(test_subsets_forced_bounds still covers it)")
    subs = _subs(name)
    assert subs, "no subset goldens"
    buf = generate_device(full["kind"], n, full["seed"])
    dev = DeviceTree()
    try:
        dev.split(buf, n, LOD_POINTS_F32, make_config(full["T"]))
        info = dev.info()
        assert [float(v).hex() for v in info.world_min] + [float(info.world_size).hex()] == full["world"]
        del buf
        gc.collect()
        torch.cuda.empty_cache()
        nodes = dev.nodes()
        _structure_properties(nodes, n, full["T"], 16)

        # skeleton at depths <= 4 (node set, kind, points in the node's cube, fp64 bounds)
        dmax = full["skeleton_depth"]
        shallow = np.flatnonzero(nodes["depth"] <= dmax)
        got = {}
        for k in shallow:
            nd = nodes[k]
            ids = subtree_index(nodes, int(nd["depth"]), nd["cell"])
            leaves = ids[(nodes["flags"][ids] & 1) == 1]
            pts = int(nodes["count"][leaves].astype(np.int64).sum())
            got[cell_path_str(nd["cell"], int(nd["depth"]))] = [
                "L" if nd["flags"] & 1 else "I", pts, [float(v).hex() for v in nd["min"]] + [float(nd["size"]).hex()]]
        bad, nbad = diff_dicts(got, full["skeleton"])
        assert nbad == 0, f"{name} skeleton: {nbad} mismatches, e.g. {bad}"

        # every golden subtree: split
        index = {}
        for g in subs:
            ids = subtree_index(nodes, g["depth"], g["cell"])
            index[g["path"]] = ids
            bad, nbad = diff_dicts(device_subtree_split(dev, nodes, ids), g["split"])
            assert nbad == 0, f"{name} subtree {g['path']}: {nbad} split mismatches, e.g. {bad}"

        # sampling: subtrees vs goldens, shallow inner nodes by induction from their children
        offender = None
        occupancy = None
        for mode in MODES:
            strat, code, seed = _mode(mode)
            errs = [g for g in subs if "error" in g["modes"][mode]]
            if strat == "random":
                exp = offender
                if errs:   # a subset's offender is deeper than any node outside the subsets
                    first = min(errs, key=lambda g: (-len(g["modes"][mode]["at"]), g["modes"][mode]["at"]))
                    assert exp is not None and exp[1] == first["modes"][mode]["at"], (exp, first["modes"][mode])
                if exp is not None:
                    with pytest.raises(ConsistencyError) as ei:
                        dev.voxelize(code, seed)
                    msg = f"{exp[0]} samples exceed the 20-bit index limit of random sampling"
                    assert str(ei.value) == msg
                    if errs:
                        assert msg == first["modes"][mode]["error"]
                    continue
            dev.voxelize(code, seed)
            nodes = dev.nodes()
            occ = _occupancy_sums(dev, nodes)   # criterion 05: occupancy is strategy-independent
            if occupancy is not None:
                assert occ == occupancy, f"{name} {mode}: occupancy differs from the other strategies"
            occupancy = occ
            if strat == "average":
                offender = _expected_offender(nodes)
            for g in subs:
                exp = g["modes"][mode]
                assert "error" not in exp, f"{name} {g['path']} {mode}: reference raised {exp}"
                bad, nbad = diff_dicts(device_subtree_voxels(dev, nodes, index[g["path"]]), exp)
                assert nbad == 0, f"{name} subtree {g['path']} {mode}: {nbad} voxel mismatches, e.g. {bad}"
            for k in np.flatnonzero((nodes["depth"] <= 2) & ((nodes["flags"] & 1) == 0)):
                c, col = _oracle_node(dev, nodes, k, strat, seed)
                gc_, gcol = decode_voxels(dev.voxel_range(int(nodes[k]["first"]), int(nodes[k]["count"])))
                p = cell_path_str(nodes[k]["cell"], int(nodes[k]["depth"]))
                assert np.array_equal(gc_, c) and np.array_equal(gcol, col), f"{name} {mode} node {p}"
    finally:
        dev.close()
        del dev
        gc.collect()
        torch.cuda.empty_cache()


def _extract_subsets(full, subs):
    """Rows of each subset (main cell inside the subset's node, input order), extracted on the
    device from the generated cloud; returns [(positions f64, colors u8, sha1(row indices))]."""
    import torch
    from paper_2302_14801_b200.device import generate_device
    n, w = full["n"], _world(full)
    lut = torch.full((256 ** 3,), -1, dtype=torch.int16)
    l3 = lut.view(256, 256, 256)
    for i, g in enumerate(subs):
        k = 8 - g["depth"]
        c = g["cell"]
        l3[c[0] << k:(c[0] + 1) << k, c[1] << k:(c[1] + 1) << k, c[2] << k:(c[2] + 1) << k] = i
    lut = lut.cuda()
    wmin = torch.tensor(w[:3], dtype=torch.float64, device="cuda")
    chunk = 1 << 27
    buf = torch.empty(chunk * 16, dtype=torch.uint8, device="cuda")
    parts = [([], []) for _ in subs]
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        generate_device(full["kind"], m, full["seed"], start=s, out=buf)
        rec = buf[:m * 16].view(m, 16)
        xyz = rec.view(torch.float32).view(m, 4)[:, :3].double()
        # reference cells_of at 256^3 (model.py:84-98): IEEE fp64 subtract, divide, *256, floor
        cell = torch.floor((xyz - wmin) / w[3] * 256.0).clamp_(0, 255).long()
        sel = lut[(cell[:, 0] * 256 + cell[:, 1]) * 256 + cell[:, 2]]
        for i in range(len(subs)):
            idx = torch.nonzero(sel == i).squeeze(1)
            if idx.numel():
                parts[i][0].append(rec[idx].cpu())
                parts[i][1].append((idx + s).cpu())
    out = []
    for recs, idx in parts:
        raw = torch.cat(recs).numpy()
        f = raw.view(np.float32).reshape(-1, 4)
        pos = f[:, :3].astype(np.float64)
        col = np.ascontiguousarray(raw.reshape(-1, 16)[:, 12:15])
        out.append((pos, col, sha(torch.cat(idx).numpy().astype(np.uint64))))
    return out


@pytest.mark.parametrize("name", FULL)
def test_subsets_forced_bounds(name):
    from paper_2302_14801_b200 import AABB, BuildConfig, ConsistencyError, PointCloud, build_lod
    from paper_2302_14801_b200.partition import Partitioner

    full = _load(os.path.join(GOLDEN, f"full_{name}.json.gz"))
    subs = _subs(name)
    w = _world(full)
    world = AABB((w[0], w[1], w[2]), w[3])
    for g, (pos, col, isha) in zip(subs, _extract_subsets(full, subs)):
        assert len(pos) == g["n"] and isha == g["index_sha"], f"{name} {g['path']}: subset extraction"
        assert sha(pos, col) == g["input_sha"]
        tree = Partitioner(PointCloud(pos, col), BuildConfig(T=g["T"]), bounds=world).run()
        pre = g["path"]
        got = {k: v for k, v in tree_split_digest(tree).items() if k.startswith(pre)}
        bad, nbad = diff_dicts(got, g["split"])
        assert nbad == 0, f"{name} {pre}: {nbad} split mismatches, e.g. {bad}"
        for mode in MODES:
            strat, _, seed = _mode(mode)
            exp = g["modes"][mode]
            if "error" in exp:
                with pytest.raises(ConsistencyError) as ei:
                    build_lod(tree, strat, seed)
                assert str(ei.value) == exp["error"]
                continue
            build_lod(tree, strat, seed)
            got = {k: v for k, v in tree_voxel_digest(tree).items() if k.startswith(pre)}
            bad, nbad = diff_dicts(got, exp)
            assert nbad == 0, f"{name} {pre} {mode}: {nbad} voxel mismatches, e.g. {bad}"
