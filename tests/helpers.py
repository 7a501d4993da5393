"""Digest helpers shared by the GPU parity tests (same format as oracle.split_digest)."""
import base64
import hashlib
import zlib

import numpy as np


def sha(*arrays):
    h = hashlib.sha1()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ps(path):
    return "".join(str(o) for o in path) or "-"


def tree_split_digest(tree):
    out = {}
    for nd in tree.iter_nodes():
        b = [float(v).hex() for v in nd.bounds.min] + [float(nd.bounds.size).hex()]
        if nd.is_leaf:
            out[ps(nd.path)] = ["L", nd.point_count, bool(nd.oversized), b,
                                sha(np.asarray(nd.point_positions, np.float64), np.asarray(nd.point_colors, np.uint8))]
        else:
            out[ps(nd.path)] = ["I", 0, False, b, ""]
    return out


def tree_voxel_digest(tree):
    return {ps(nd.path): [nd.voxel_count, sha(nd.voxel_coords, nd.voxel_colors)] for nd in tree.inner_nodes()}


def diff_dicts(got, exp, limit=8):
    keys = sorted(set(got) | set(exp))
    bad = [(k, got.get(k), exp.get(k)) for k in keys if got.get(k) != exp.get(k)]
    return bad[:limit], len(bad)


def weighted_colors(entry):
    """Decode a golden "weighted" entry [m, sha1(coords), b64(zlib(colors))] -> (m, sha, (m,3) u8)."""
    m, csha, blob = entry
    cols = np.frombuffer(zlib.decompress(base64.b64decode(blob)), np.uint8).reshape(-1, 3)
    return m, csha, cols


def compare_weighted(got, exp):
    """got: path-string -> (coords, colors).  Coordinates must match exactly, colours within
    +-1 per channel (SPEC.md "Weighted accumulation order").  Returns (errors, n_off_by_one,
    n_channels)."""
    errors, off, total = [], 0, 0
    if set(got) != set(exp):
        errors.append(("node set", sorted(set(got) ^ set(exp))[:4]))
        return errors, off, total
    for k, entry in exp.items():
        m, csha, ecol = weighted_colors(entry)
        c, col = got[k]
        if len(c) != m or sha(c) != csha:
            errors.append((k, "coords"))
            continue
        d = np.abs(np.asarray(col, np.int16) - ecol.astype(np.int16))
        total += d.size
        off += int((d == 1).sum())
        if d.max(initial=0) > 1:
            errors.append((k, "colour off by", int(d.max())))
    return errors, off, total


def cell_path_str(cell, depth):
    cx, cy, cz = (int(c) for c in cell)
    return "".join(str(((cx >> b) & 1) | (((cy >> b) & 1) << 1) | (((cz >> b) & 1) << 2))
                   for b in range(depth - 1, -1, -1)) or "-"


def subtree_index(nodes, depth, cell):
    """Node-table ids of the subtree rooted at (depth, cell), vectorised over the table."""
    d = nodes["depth"].astype(np.int64)
    c = nodes["cell"].astype(np.int64)
    sh = np.maximum(d - depth, 0)[:, None]
    inside = (d >= depth) & np.all((c >> sh) == np.asarray(cell, np.int64)[None, :], axis=1)
    return np.flatnonzero(inside)


def device_subtree_split(dev, nodes, ids):
    """Split digests (make_golden format) of node ids, reading only those nodes' points."""
    from paper_2302_14801_b200.device import unpack_records
    fmt = dev.info().point_format
    out = {}
    for k in ids:
        nd = nodes[k]
        b = [float(v).hex() for v in nd["min"]] + [float(nd["size"]).hex()]
        p = cell_path_str(nd["cell"], int(nd["depth"]))
        if nd["flags"] & 1:
            pos, col = unpack_records(dev.leaf_range(int(nd["first"]), int(nd["count"])), fmt)
            out[p] = ["L", int(nd["count"]), bool(nd["flags"] & 2), b, sha(pos, col)]
        else:
            out[p] = ["I", 0, False, b, ""]
    return out


def decode_voxels(raw):
    key, rgb = raw[:, 0], raw[:, 1]
    coords = np.stack([key >> 14, (key >> 7) & 127, key & 127], axis=1).astype(np.uint8)
    colors = np.stack([rgb & 255, (rgb >> 8) & 255, (rgb >> 16) & 255], axis=1).astype(np.uint8)
    return coords, colors


def device_subtree_voxels(dev, nodes, ids):
    """Voxel digests [m, sha1(coords || colors)] of the inner nodes among `ids`."""
    out = {}
    for k in ids:
        nd = nodes[k]
        if nd["flags"] & 1:
            continue
        c, col = decode_voxels(dev.voxel_range(int(nd["first"]), int(nd["count"])))
        out[cell_path_str(nd["cell"], int(nd["depth"]))] = [int(nd["count"]), sha(c, col)]
    return out
