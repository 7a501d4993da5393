"""GPU edge cases checked directly against the CPU oracle (oracle/lod_oracle.py, itself
pinned to the reference's goldens):

* a voxel with > 65793 samples of colour 255: its colour sum passes 2^24, so the f32
  vector reductions of the average path must hand over to exact u64 sums;
* duplicate points forming an oversized leaf at max depth, under every strategy."""
import numpy as np
import pytest

from oracle import lod_oracle as O

pytestmark = pytest.mark.gpu


def _cloud(n_dup, n_rest, seed=0):
    rng = np.random.default_rng(seed)
    dup = np.tile([[0.3125, 0.625, 0.8125]], (n_dup, 1))
    rest = rng.random((n_rest, 3))
    pos = np.concatenate([dup, rest]).astype(np.float32).astype(np.float64)
    col = np.concatenate([np.full((n_dup, 3), 255, np.uint8), rng.integers(0, 256, (n_rest, 3)).astype(np.uint8)])
    perm = rng.permutation(len(pos))
    return pos[perm], col[perm]


def _compare(pos, col, T, strategy, seed=0):
    from paper_2302_14801_b200 import BuildConfig, PointCloud, build_lod, partition
    tree = partition(PointCloud(pos, col), BuildConfig(T=T))
    build_lod(tree, strategy, seed)
    sp = O.split(pos, T=T)
    vox = O.voxelize(sp, pos, col, strategy, seed)
    got = {nd.path: nd for nd in tree.iter_nodes()}
    assert set(got) == set(sp.nodes)
    for path, (c, k) in vox.items():
        g = got[path]
        if strategy == "weighted":
            assert np.array_equal(g.voxel_coords, c)
            assert np.abs(g.voxel_colors.astype(int) - k.astype(int)).max(initial=0) <= 1
        else:
            assert np.array_equal(g.voxel_coords, c) and np.array_equal(g.voxel_colors, k), (strategy, path)
    return tree


def test_average_sum_overflow_falls_back_to_exact():
    pos, col = _cloud(70_000, 30_000)
    tree = _compare(pos, col, 1000, "average")
    over = [nd for nd in tree.leaves() if nd.oversized]
    assert over and max(nd.point_count for nd in over) == 70_000


def test_average_exact_sums_past_2_32():
    """17M coincident samples of colour 255 in one voxel: the channel sums (4.3e9) pass 2^32,
    so the exact fallback must keep full u64 sums per channel (the reference sums in int64,
    sampling.py:92-96)."""
    pos, col = _cloud(17_000_000, 30_000)
    tree = _compare(pos, col, 1000, "average")
    over = [nd for nd in tree.leaves() if nd.oversized]
    assert over and max(nd.point_count for nd in over) == 17_000_000


@pytest.mark.parametrize("strategy", ["first-come", "random", "weighted"])
def test_oversized_duplicates_all_strategies(strategy):
    pos, col = _cloud(3_000, 20_000, seed=1)
    _compare(pos, col, 500, strategy, seed=4)


def test_distribute_two_pass_leaf_id_path():
    """> 2^19 leaves: the 2nd radix digit no longer fits the f32 record pad, so the
    distribute carries leaf ids in a separate array (distribute.cu OUT_LEAF)."""
    from paper_2302_14801_b200 import BuildConfig, PointCloud, partition
    rng = np.random.default_rng(11)
    pos = rng.random((2_500_000, 3)).astype(np.float32).astype(np.float64)
    col = rng.integers(0, 256, (len(pos), 3)).astype(np.uint8)
    tree = partition(PointCloud(pos, col), BuildConfig(T=3))
    info = tree.device_tree.info()
    assert info.n_leaves > (1 << 19) and info.radix_passes == 2
    sp = O.split(pos, T=3)
    got = {nd.path: nd for nd in tree.leaves()}
    exp = {p: nd for p, nd in sp.nodes.items() if nd.kind == "leaf"}
    assert set(got) == set(exp)
    rng2 = np.random.default_rng(0)
    for path in rng2.choice(len(exp), 2000, replace=False):
        p = list(exp)[path]
        assert np.array_equal(got[p].point_positions, pos[exp[p].idx]), p
