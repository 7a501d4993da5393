"""Digest helpers shared by the GPU parity tests (same format as oracle.split_digest)."""
import hashlib

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
