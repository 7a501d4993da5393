"""Stage-level goldens from the REAL reference Partitioner (build container only):

    python tests/golden/make_stage_golden.py  -> tests/golden/stages.json.gz

For each case of STAGE_CASES the reference's `Partitioner(cloud, cfg)` stages are run one at a
time (partition.py:99-287) and their intermediate values digested: the count grid, the
extension tree (per ExtendedPyramid: anchor path / cell, depth, finest counts, point_idx,
rel_cells), the merged pyramid levels of every tier and the leaf list (path, count) in the
reference's leaf numbering.  tests/test_oracle_golden.py pins the oracle's tiers to these;
the GPU stage tests (tests/test_gpu_stages.py) hold the device to the oracle.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from stage_cases import STAGE_CASES, case_name, custom_cloud  # noqa: E402


def stage_cloud(kind, n, seed):
    from lodforge.ingest import GeneratorPreset, PointCloud, generate
    arrays = custom_cloud(kind, n, seed)
    if arrays is not None:
        return PointCloud(*arrays)
    return generate(GeneratorPreset(kind, n, seed))


def sha(a) -> str:
    return hashlib.sha1(np.ascontiguousarray(np.asarray(a, np.int64)).tobytes()).hexdigest()


def digest_ext(ep, levels_attr="levels") -> dict:
    return {
        "anchor_path": list(ep.anchor_path), "anchor_cell": [int(v) for v in ep.anchor_cell], "depth": int(ep.depth),
        "finest": sha(ep.finest), "point_idx": sha(ep.point_idx), "rel_cells": sha(ep.rel_cells),
        "levels": [sha(l) for l in getattr(ep, levels_attr)],
        "children": {",".join(map(str, k)): digest_ext(c, levels_attr) for k, c in sorted(ep.children.items())},
    }


def main():
    from lodforge.model import BuildConfig
    from lodforge.partition import Partitioner
    out = {}
    for kind, n, seed, cfg in STAGE_CASES:
        p = Partitioner(stage_cloud(kind, n, seed), BuildConfig(**cfg))
        grid = p.count()
        p.extend_overfull_cells()
        levels = p.merge()
        p.build_targets()
        p.insert()
        out[case_name(kind, n, seed, cfg)] = {
            "grid": sha(grid), "grid_sum": int(grid.sum()),
            "levels": [sha(l) for l in levels],
            "extended": {",".join(map(str, k)): digest_ext(ep) for k, ep in sorted(p.extended.items())},
            "leaves": [[list(nd.path), int(c)] for nd, c in zip(p.leaf_nodes, p.leaf_counts)],
        }
        print(kind, n, cfg, len(p.extended), sum(1 for _ in p._iter_extended()), len(p.leaf_nodes))
    with gzip.open(os.path.join(HERE, "stages.json.gz"), "wt") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
