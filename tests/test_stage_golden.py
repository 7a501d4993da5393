"""Pin the oracle's stage values (oracle/lod_oracle.py split tiers) to the REAL reference's
Partitioner stages (tests/golden/stages.json.gz from make_stage_golden.py): count grid,
extension tree (anchor, depth, finest counts, member points, relative cells), merged pyramids
of every tier and the leaf set.  The GPU stage tests hold the device to the same digests."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden
from stage_cases import STAGE_CASES, case_name, custom_cloud
from oracle import lod_oracle as O


def sha(a):
    return hashlib.sha1(np.ascontiguousarray(np.asarray(a, np.int64)).tobytes()).hexdigest()


def cloud_arrays(kind, n, seed):
    arrays = custom_cloud(kind, n, seed)
    if arrays is not None:
        return arrays
    from paper_2302_14801_b200.generators import reference_cloud
    c = reference_cloud(kind, n, seed)
    return c.positions, c.colors


def tier_digest(t):
    return {
        "anchor_path": list(t.prefix), "anchor_cell": [int(v) for v in t.anchor], "depth": int(t.levels_n),
        "finest": sha(t.counts), "point_idx": sha(t.idx), "rel_cells": sha(t.fine),
        "levels": [sha(l) for l in t.levels],
        "children": {",".join(map(str, k)): tier_digest(c) for k, c in sorted(t.subs.items())},
    }


@pytest.mark.parametrize("case", STAGE_CASES, ids=[case_name(*c) for c in STAGE_CASES])
def test_oracle_stages_match_reference(case):
    kind, n, seed, cfg = case
    g = load_golden("stages")[case_name(*case)]
    pos, _ = cloud_arrays(kind, n, seed)
    full = dict(T=50_000, initial_depth=8, extension_depth=4, max_depth=16, **{})
    full.update(cfg)
    sp = O.split(pos, **full)
    top = sp.top
    assert sha(top.counts) == g["grid"] and int(top.counts.sum()) == g["grid_sum"]
    assert [sha(l) for l in top.levels] == g["levels"]
    assert {",".join(map(str, k)): tier_digest(t) for k, t in sorted(top.subs.items())} == g["extended"]
    leaves = {tuple(p): c for p, c in g["leaves"]}
    assert {p: nd.count for p, nd in sp.nodes.items() if nd.kind == "leaf"} == leaves
