"""CPU checks of the large-config parity machinery (no GPU):

* the C restatement of the synthetic generators (`oracle/synth.c`, used to scan the 500M-4B
  point clouds for the subtree-subset goldens and the CPU baseline) is bit-identical to the
  numpy generators (and so to the device generator, tests/test_gpu_generators.py);
* the subtree-subset method itself (probe 6): the oracle's split + sampling of
  the points inside an inner node with the full cloud's bounds forced reproduce the full
  build's subtree at that node, for every strategy;
* the committed large-config goldens are mutually consistent.
"""
import glob
import gzip
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import cell_path_str
from oracle import lod_oracle as O
from oracle.synth import Cloud, subtree_subset, world_of
from paper_2302_14801_b200.generators import synthetic_rows

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("kind,seed", [("sphere", 1), ("terrain", 2), ("scene", 3), ("cluster", 4), ("surface", 5)])
def test_c_generator_matches_numpy(kind, seed):
    c = Cloud(kind, seed)
    for start in (0, 123_456_789, 3_999_990_000):
        p, col = c.rows(start, 5000)
        p2, col2 = synthetic_rows(kind, seed, start, 5000)
        assert np.array_equal(p.view(np.uint32), p2.view(np.uint32)), (kind, start)
        assert np.array_equal(col, col2), (kind, start)
    idx = np.array([7, 5, 10**9 + 3, 17], np.uint64)
    p, col = c.rows_idx(idx)
    for i, r in enumerate(idx):
        p2, col2 = synthetic_rows(kind, seed, int(r), 1)
        assert np.array_equal(p[i], p2[0]) and np.array_equal(col[i], col2[0])


def test_world_of_matches_reference_rule():
    c = Cloud("scene", 3)
    lo, size = world_of(c, 300_000, chunk=70_000)
    pos, _ = synthetic_rows("scene", 3, 0, 300_000)
    lo2, size2 = O.world_bounds(pos.astype(np.float64))
    assert tuple(lo) == lo2 and size == size2


@pytest.mark.parametrize("strategy", ["average", "random", "first-come"])
def test_subtree_subset_reproduces_full_subtree(strategy):
    """Partitioner(subset, cfg, bounds=world) == the full tree's subtree (probe 6)."""
    kind, n, seed, T = "cluster", 300_000, 4, 2000
    sub = subtree_subset(kind, n, seed, target=40_000, T=T, chunk=100_000)
    pos, _ = synthetic_rows(kind, seed, 0, n)
    pos = pos.astype(np.float64)
    _, col = synthetic_rows(kind, seed, 0, n)
    full = O.split(pos, T=T)
    fvox = O.voxelize(full, pos, col, strategy, 1)
    part = O.split(sub["positions"], T=T, bounds=sub["world"])
    pvox = O.voxelize(part, sub["positions"], sub["colors"], strategy, 1)
    pre = cell_path_str(sub["cell"], sub["depth"])
    fd = {k: v for k, v in O.split_digest(full, pos, col).items() if k.startswith(pre)}
    pd = {k: v for k, v in O.split_digest(part, sub["positions"], sub["colors"]).items() if k.startswith(pre)}
    assert fd and fd == pd
    fv = {k: v for k, v in O.voxel_digest(fvox).items() if k.startswith(pre)}
    pv = {k: v for k, v in O.voxel_digest(pvox).items() if k.startswith(pre)}
    assert fv and fv == pv


FULL = sorted(glob.glob(os.path.join(GOLDEN, "full_*.json.gz")))


def _load(fn):
    with gzip.open(fn, "rt") as f:
        return json.load(f)


@pytest.mark.parametrize("fn", FULL, ids=[os.path.basename(f) for f in FULL])
def test_large_goldens_consistent(fn):
    full = _load(fn)
    name = full["config"]
    subs = [_load(f) for f in sorted(glob.glob(os.path.join(GOLDEN, f"sub_{name}_*.json.gz")))]
    assert sorted(g["path"] for g in subs) == sorted(full["subsets"])
    assert full["skeleton"]["-"][1] == full["n"]
    for g in subs:
        assert g["world"] == full["world"] and g["n_full"] == full["n"]
        assert g["path"] in g["split"] and g["split"][g["path"]][0] == "I"
        # the subset's leaves hold exactly its points
        assert sum(v[1] for v in g["split"].values() if v[0] == "L") == g["n"]
        # nodes the skeleton also lists agree on kind, count (points in the cube) and bounds
        for p, v in g["split"].items():
            if p in full["skeleton"]:
                kind, cnt, b = full["skeleton"][p]
                assert v[0] == kind and v[3] == b
                if kind == "L":
                    assert v[1] == cnt
        for mode, exp in g["modes"].items():
            if "error" in exp:
                assert exp["error"].endswith("samples exceed the 20-bit index limit of random sampling")
                assert exp["at"].startswith(g["path"])


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not present")
def test_exceptions_are_the_reference_classes_when_importable():
    code = ("import sys; sys.path.insert(0, '/root/reference/pkg/src'); import lodforge.errors as E; "
            "import paper_2302_14801_b200 as P; "
            "assert P.ConsistencyError is E.ConsistencyError and P.FormatError is E.FormatError; print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, PYTHONPATH=root))
    assert r.stdout.strip() == "ok", r.stderr
