"""The reference's per-node sampling helpers on the device (sampling.py:21-160):
project_child_samples, extract_first_come / _random / _average / _weighted and sample_*.

Ports reference tests/test_sampling.py TestProjection / TestFirstCome / TestRandom /
TestAverage / TestWeighted, then holds the device helpers to the oracle's restatement
(oracle/lod_oracle.py extract_*, child_gpos) on random sample lists and on real trees:
bit-exact for first-come / random / average and the projection, +-1 per channel for weighted
(the reference's own tolerance against its oracle, test_sampling.py:234)."""
import numpy as np
import pytest

from oracle import lod_oracle as orc

pytestmark = pytest.mark.gpu


def _S():
    from paper_2302_14801_b200 import sampling
    return sampling


def _tree(n=20_000, T=2000, kind="uniform-cube", seed=1, strategy="first-come"):
    from paper_2302_14801_b200 import BuildConfig, build_lod, partition
    from paper_2302_14801_b200.generators import reference_cloud
    cloud = reference_cloud(kind, n, seed)
    tree = partition(cloud, BuildConfig(T=T))
    if strategy:
        build_lod(tree, strategy, 0)
    return cloud, tree


# -------------------------------------------------------------------------- TestProjection
def test_projection_inner_child_voxel_offsets():
    _, tree = _tree()
    node = next(n for n in tree.inner_nodes() if any(not c.is_leaf for _, c in n.existing_children()))
    gpos, _ = _S().project_child_samples(node)
    assert (gpos >= 0).all() and (gpos < 128).all()


def test_projection_max_face_point_clamps_to_last_cell():
    from paper_2302_14801_b200 import BuildConfig, PointCloud, partition
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]] * 600)
    tree = partition(PointCloud(pos, np.zeros((len(pos), 3), np.uint8)), BuildConfig(T=1000))
    assert not tree.root.is_leaf
    gpos, _ = _S().project_child_samples(tree.root)
    assert gpos.max() < 128 and np.floor(gpos).max() == 127


def test_projection_of_leaf_raises():
    _, tree = _tree(strategy=None)
    with pytest.raises(ValueError):
        _S().project_child_samples(tree.leaves()[0])


def test_projection_equals_oracle_every_inner_node():
    """Leaf children: clip((p - min) / size * 128); voxel children: octant offset + (c + .5) / 2."""
    cloud, tree = _tree(n=60_000, T=1500, kind="stadium", seed=3)
    for node in tree.inner_nodes():
        gpos, cols = _S().project_child_samples(node)
        lo = node.bounds.min_array()
        gp, cc = [], []
        for o, ch in node.existing_children():
            if ch.is_leaf:
                gp.append(np.clip((ch.point_positions - lo) / node.bounds.size * 128.0, 0.0, np.nextafter(128.0, 0)))
                cc.append(ch.point_colors)
            else:
                off = np.array([64.0 * (o & 1), 64.0 * ((o >> 1) & 1), 64.0 * ((o >> 2) & 1)])
                gp.append(off + (ch.voxel_coords.astype(np.float64) + 0.5) / 2.0)
                cc.append(ch.voxel_colors)
        assert np.array_equal(gpos, np.concatenate(gp)) and np.array_equal(cols, np.concatenate(cc))


# ---------------------------------------------------------------------------- TestFirstCome
def test_first_come_smallest_ordinal_wins():
    coords, out = _S().extract_first_come(np.array([[5.2, 5.2, 5.2], [5.8, 5.8, 5.8]]),
                                          np.array([[10, 0, 0], [20, 0, 0]], np.uint8))
    assert len(coords) == 1 and tuple(out[0]) == (10, 0, 0)


def test_first_come_constant_color_preserved():
    gpos = np.random.default_rng(0).random((500, 3)) * 128
    _, out = _S().extract_first_come(gpos, np.full((500, 3), 77, np.uint8))
    assert (out == 77).all()


def test_first_come_output_ordered_by_winner_ordinal():
    coords, out = _S().extract_first_come(np.array([[100.5, 0.5, 0.5], [3.5, 3.5, 3.5], [100.5, 0.5, 0.5]]),
                                          np.array([[1, 1, 1], [2, 2, 2], [3, 3, 3]], np.uint8))
    assert tuple(out[0]) == (1, 1, 1) and tuple(out[1]) == (2, 2, 2)


# ------------------------------------------------------------------------------ TestRandom
def test_random_sample_count_limit():
    from paper_2302_14801_b200.errors import ConsistencyError
    n = 1 << 20
    with pytest.raises(ConsistencyError):
        _S().extract_random(np.zeros((n, 3)), np.zeros((n, 3), np.uint8), 0, 0)


def test_random_deterministic_and_tie_prefers_larger_ordinal():
    g = np.tile(np.array([[7.5, 7.5, 7.5]]), (4, 1))
    c = np.arange(12, dtype=np.uint8).reshape(4, 3)
    a = _S().extract_random(g, c, 9, 123)
    b = _S().extract_random(g, c, 9, 123)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    e = orc.extract_random(np.floor(g).astype(np.int64), c, 9, 123)
    assert np.array_equal(a[1], e[1])


# ----------------------------------------------------------------------------- TestAverage
def test_average_arithmetic_mean_and_half_away_from_zero():
    g = np.array([[5.1, 5.1, 5.1], [5.9, 5.9, 5.9]])
    assert tuple(_S().extract_average(g, np.array([[200, 0, 0], [100, 0, 0]], np.uint8))[1][0]) == (150, 0, 0)
    assert tuple(_S().extract_average(g, np.array([[200, 0, 0], [101, 0, 0]], np.uint8))[1][0]) == (151, 0, 0)


# ---------------------------------------------------------------------------- TestWeighted
def test_weighted_sample_at_cell_center_keeps_own_color():
    coords, out = _S().extract_weighted(np.array([[10.5, 10.5, 10.5]]), np.array([[40, 80, 120]], np.uint8))
    assert len(coords) == 1 and tuple(coords[0]) == (10, 10, 10) and tuple(out[0]) == (40, 80, 120)


def test_weighted_non_occupied_neighbors_not_emitted():
    coords, _ = _S().extract_weighted(np.array([[10.9, 10.9, 10.9]]), np.array([[50, 50, 50]], np.uint8))
    assert {tuple(c) for c in coords.tolist()} == {(10, 10, 10)}


# ------------------------------------------------------------------- oracle on random lists
def _samples(S, seed, spread):
    rng = np.random.default_rng(seed)
    if spread == "dense":       # few cells, many samples per cell
        g = rng.random((S, 3)) * 4 + 60
    elif spread == "grid":      # exact cell boundaries and the 127 face
        g = rng.integers(0, 256, (S, 3)) / 2.0
        g[: S // 50] = np.nextafter(128.0, 0)
    else:
        g = rng.random((S, 3)) * 128
    return np.minimum(g, np.nextafter(128.0, 0)), rng.integers(0, 256, (S, 3)).astype(np.uint8)


@pytest.mark.parametrize("S", [1, 31, 1000, 100_000, (1 << 20) - 1])
@pytest.mark.parametrize("spread", ["uniform", "dense", "grid"])
def test_extract_equals_oracle(S, spread):
    g, c = _samples(S, S + len(spread), spread)
    cells = np.floor(g).astype(np.int64)
    for name in ("first_come", "average"):
        got = getattr(_S(), f"extract_{name}")(g, c)
        exp = getattr(orc, f"extract_{name}")(cells, c)
        assert np.array_equal(got[0], exp[0]) and np.array_equal(got[1], exp[1]), name
    for seed, h in ((0, 0), (7, 0x1234567890ABCDEF)):
        got = _S().extract_random(g, c, seed, h)
        exp = orc.extract_random(cells, c, seed, h)
        assert np.array_equal(got[0], exp[0]) and np.array_equal(got[1], exp[1])
    if S <= 100_000:
        got = _S().extract_weighted(g, c)
        exp = orc.extract_weighted(g, c)
        assert np.array_equal(got[0], exp[0])
        assert np.abs(got[1].astype(int) - exp[1].astype(int)).max(initial=0) <= 1


def test_extract_empty_and_outside_grid():
    z = np.zeros((0, 3))
    for name in ("first_come", "average", "weighted"):
        co, cl = getattr(_S(), f"extract_{name}")(z, np.zeros((0, 3), np.uint8))
        assert co.shape == (0, 3) and cl.shape == (0, 3)
    with pytest.raises(ValueError):
        _S().extract_average(np.array([[128.0, 0.0, 0.0]]), np.zeros((1, 3), np.uint8))


# ------------------------------------------------------------- sample_* on a built tree
@pytest.mark.parametrize("strategy", ["first-come", "random", "average", "weighted"])
def test_sample_node_equals_build(strategy):
    """sample_<strategy>(node) on a built tree reproduces the node's voxels from build_lod."""
    from paper_2302_14801_b200 import rng
    _, tree = _tree(n=60_000, T=1500, kind="stadium", seed=3, strategy=strategy)
    S = _S()
    for node in tree.inner_nodes():
        if strategy == "random":
            co, cl = S.sample_random(node, 0)
            g, c = S.project_child_samples(node)
            e = orc.extract_random(np.floor(g).astype(np.int64), c, 0, rng.path_hash(0, node.path))
            assert np.array_equal(co, e[0]) and np.array_equal(cl, e[1])
        else:
            co, cl = getattr(S, "sample_" + strategy.replace("-", "_"))(node)
        assert np.array_equal(co, node.voxel_coords)
        if strategy == "weighted":
            assert np.abs(cl.astype(int) - node.voxel_colors.astype(int)).max(initial=0) <= 1
        else:
            assert np.array_equal(cl, node.voxel_colors)
