"""The reference's stage-level split API on the device (partition.py:36-297): `merge_pyramid`
and the Partitioner stages count / extend_overfull_cells / merge / build_targets / insert.

Ports reference tests/test_partition.py TestCount and TestMergePyramid, then holds every
stage's intermediate value to the oracle's tiers (oracle/lod_oracle.py split: counts, the
extension tree with its member points and relative cells, the merged pyramids) and the final
tree to the oracle's leaves."""
import numpy as np
import pytest

from oracle import lod_oracle as orc

pytestmark = pytest.mark.gpu

UNMERGEABLE = 0xFFFFFFFF


def _uniform(n, seed=42):
    from paper_2302_14801_b200.generators import reference_cloud
    return reference_cloud("uniform-cube", n, seed)


# ---------------------------------------------------------------------------- TestCount
def test_count_conservation():
    from paper_2302_14801_b200 import BuildConfig
    from paper_2302_14801_b200.partition import Partitioner
    grid = Partitioner(_uniform(100_000), BuildConfig()).count()
    assert grid.shape == (256, 256, 256) and grid.dtype == np.int64
    assert grid.sum() == 100_000


def test_count_degenerate_cluster():
    from paper_2302_14801_b200 import AABB, BuildConfig, PointCloud
    from paper_2302_14801_b200.partition import Partitioner
    n = 500
    cloud = PointCloud(np.zeros((n, 3)), np.zeros((n, 3), np.uint8))
    grid = Partitioner(cloud, BuildConfig(), bounds=AABB((0, 0, 0), 1)).count()
    assert grid[0, 0, 0] == n and grid.sum() == n


def test_count_matches_brute_force_histogram():
    from paper_2302_14801_b200 import BuildConfig
    from paper_2302_14801_b200.partition import Partitioner
    cloud = _uniform(1000)
    p = Partitioner(cloud, BuildConfig())
    grid = p.count()
    lo, size = orc.world_bounds(cloud.positions)
    cells = orc.grid_cells(cloud.positions, lo, size, 256)
    expected = np.zeros((256, 256, 256), np.int64)
    np.add.at(expected, tuple(cells.T), 1)
    assert np.array_equal(grid, expected)
    assert np.array_equal(p.cells, cells)
    assert p.bounds.size == size and tuple(p.bounds.min) == tuple(lo)


def test_count_point_outside_forced_bounds_raises():
    from paper_2302_14801_b200 import AABB, BuildConfig, PointCloud
    from paper_2302_14801_b200.errors import ConsistencyError
    from paper_2302_14801_b200.partition import Partitioner
    pos = np.random.default_rng(0).random((1000, 3))
    pos[10] = (2.0, 0.5, 0.5)
    with pytest.raises(ConsistencyError):
        Partitioner(PointCloud(pos, np.zeros((1000, 3), np.uint8)), BuildConfig(), bounds=AABB((0, 0, 0), 1)).count()


# ---------------------------------------------------------------------- TestMergePyramid
def _grid(dim, entries):
    g = np.zeros((dim, dim, dim), np.int64)
    for cell, v in entries.items():
        g[cell] = v
    return g


def test_merge_small_group_merges():
    from paper_2302_14801_b200.partition import merge_pyramid
    levels = merge_pyramid(_grid(2, {(x, y, z): 1000 for x in (0, 1) for y in (0, 1) for z in (0, 1)}), T=50_000)
    assert levels[0].flat[0] == 8000 and (levels[1] == 0).all()


def test_merge_group_at_threshold_flags_parent():
    from paper_2302_14801_b200.partition import merge_pyramid
    levels = merge_pyramid(_grid(2, {(0, 0, 0): 49_999, (1, 0, 0): 1}), T=50_000)
    assert levels[0].flat[0] == UNMERGEABLE
    assert levels[1][0, 0, 0] == 49_999 and levels[1][1, 0, 0] == 1


def test_merge_unmergeable_child_propagates():
    from paper_2302_14801_b200.partition import merge_pyramid
    levels = merge_pyramid(_grid(2, {(0, 0, 0): UNMERGEABLE, (1, 1, 1): 3}), T=50_000)
    assert levels[0].flat[0] == UNMERGEABLE and levels[1][1, 1, 1] == 3


def test_merge_empty_group_stays_empty():
    from paper_2302_14801_b200.partition import merge_pyramid
    assert merge_pyramid(np.zeros((4, 4, 4), np.int64), T=10)[0].flat[0] == 0


def test_merge_cascade_over_two_levels():
    from paper_2302_14801_b200.partition import merge_pyramid
    levels = merge_pyramid(_grid(4, {(0, 0, 0): 5, (3, 3, 3): 7}), T=100)
    assert levels[0].flat[0] == 12 and (levels[1] == 0).all() and (levels[2] == 0).all()


@pytest.mark.parametrize("dim,T,seed", [(1, 5, 0), (2, 3, 1), (8, 40, 2), (32, 200, 3), (64, 5000, 4), (256, 50_000, 5)])
def test_merge_random_grids_equal_oracle(dim, T, seed):
    from paper_2302_14801_b200.partition import merge_pyramid
    rng = np.random.default_rng(seed)
    finest = rng.integers(0, max(2, T // 4), (dim, dim, dim)).astype(np.int64)
    finest[rng.random(finest.shape) < 0.5] = 0
    finest[rng.random(finest.shape) < 0.01] = UNMERGEABLE
    finest[rng.random(finest.shape) < 0.005] = T + 7   # overfull plain counts
    got = merge_pyramid(finest, T)
    exp = orc.merge_levels(finest, T)
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        assert np.array_equal(g, e)


def test_merge_rejects_bad_grids():
    from paper_2302_14801_b200.partition import merge_pyramid
    with pytest.raises(ValueError):
        merge_pyramid(np.zeros((3, 3, 3), np.int64), 10)
    with pytest.raises(ValueError):
        merge_pyramid(np.full((2, 2, 2), 1 << 40, np.int64), 10)


# ----------------------------------------------- stages vs the reference's stage goldens
def _ep_digest(ep):
    from test_stage_golden import sha
    return {
        "anchor_path": list(ep.anchor_path), "anchor_cell": [int(v) for v in ep.anchor_cell], "depth": int(ep.depth),
        "finest": sha(ep.finest), "point_idx": sha(ep.point_idx), "rel_cells": sha(ep.rel_cells),
        "levels": [sha(l) for l in ep.levels],
        "children": {",".join(map(str, k)): _ep_digest(c) for k, c in ep.children.items()},
    }


def _same(got, exp, where):
    """Recursive equality naming the first differing field."""
    if isinstance(exp, dict):
        assert isinstance(got, dict) and set(got) == set(exp), f"{where}: keys {sorted(got)} != {sorted(exp)}"
        for k in exp:
            _same(got[k], exp[k], f"{where}.{k}")
    else:
        assert got == exp, f"{where}: {got} != {exp}"


def _cloud(kind, n, seed):
    from paper_2302_14801_b200 import PointCloud
    from test_stage_golden import cloud_arrays
    return PointCloud(*cloud_arrays(kind, n, seed))


from stage_cases import STAGE_CASES, case_name  # noqa: E402


@pytest.mark.parametrize("case", STAGE_CASES, ids=[case_name(*c) for c in STAGE_CASES])
def test_stages_equal_reference(case):
    """Every stage's value equals the reference Partitioner's (digests in stages.json.gz; the
    dict orders and the leaf numbering too), and the inserted leaves equal the oracle's."""
    from paper_2302_14801_b200 import BuildConfig
    from paper_2302_14801_b200.partition import Partitioner
    from test_stage_golden import sha
    from conftest import load_golden
    kind, n, seed, cfg = case
    g = load_golden("stages")[case_name(*case)]
    cloud = _cloud(kind, n, seed)
    p = Partitioner(cloud, BuildConfig(**cfg))
    grid = p.count()
    assert sha(grid) == g["grid"] and int(grid.sum()) == g["grid_sum"]
    ext = p.extend_overfull_cells()
    levels = p.merge()
    assert [sha(l) for l in levels] == g["levels"]
    _same({",".join(map(str, k)): _ep_digest(ep) for k, ep in ext.items()}, g["extended"], "extended")
    assert list(g["extended"]) == [",".join(map(str, k)) for k in ext]     # reference dict order
    tree = p.build_targets()
    assert [[list(nd.path), c] for nd, c in zip(p.leaf_nodes, p.leaf_counts)] == g["leaves"]
    for lvl, ref in zip(p.levels, p.refs):   # refs point at the leaf of each plain cell
        flat = lvl.reshape(-1)
        assert np.array_equal(ref >= 0, (flat != 0) & (flat != UNMERGEABLE))
        assert np.array_equal(np.asarray(p.leaf_counts)[ref[ref >= 0]], flat[ref >= 0])
    p.insert()
    full = dict(T=50_000, initial_depth=8, extension_depth=4, max_depth=16)
    full.update(cfg)
    sp = orc.split(cloud.positions, **full)
    for leaf in p.leaf_nodes:
        exp = sp.nodes[leaf.path]
        assert leaf.oversized == exp.oversized
        assert np.array_equal(leaf.point_positions, cloud.positions[exp.idx])
        assert np.array_equal(leaf.point_colors, cloud.colors[exp.idx])
    assert tree.root is p.nodes[()]


def test_stages_order_and_run_completion():
    from paper_2302_14801_b200 import BuildConfig, partition
    from paper_2302_14801_b200.partition import Partitioner
    cloud = _cloud("blobs", 150_000, 11)
    p = Partitioner(cloud, BuildConfig(T=500))
    with pytest.raises(RuntimeError):
        p.merge()
    p.count()
    with pytest.raises(RuntimeError):
        p.count()
    tree = p.run()             # finishes the remaining stages
    ref = partition(cloud, BuildConfig(T=500))
    a = sorted((lf.path, lf.point_count) for lf in tree.leaves())
    b = sorted((lf.path, lf.point_count) for lf in ref.leaves())
    assert a == b
    # a tree built stage by stage samples like the fused build
    from paper_2302_14801_b200 import build_lod
    for strategy, seed in (("average", 0), ("random", 5)):
        build_lod(tree, strategy, seed)
        build_lod(ref, strategy, seed)
        va = {n.path: (n.voxel_coords.tobytes(), n.voxel_colors.tobytes()) for n in tree.inner_nodes()}
        vb = {n.path: (n.voxel_coords.tobytes(), n.voxel_colors.tobytes()) for n in ref.inner_nodes()}
        assert va == vb, strategy
