"""Error paths of the drop-in vs the reference's exceptions and messages (SURVEY 8(b) "Errors").

Every message below is the reference's text, at the cited line:
  ValueError
    cannot partition an empty point cloud                 partition.py:83-84
    point coordinates must be finite                      model.py:202-205 (world_bounds_of)
    T must be >= 1 / max_depth must be >= initial_depth / max_depth must be <= 16
                                                          model.py:118-124 (BuildConfig)
    unknown sampling strategy: X                          sampling.py:169-170
    positions/colors length mismatch                      ingest.py:29-31 (PointCloud)
  ConsistencyError
    point outside bounds during grid projection           model.py:93-95 (forced bounds, partition.py:87)
    {S} samples exceed the 20-bit index limit ...         sampling.py:73-75 (covered by the goldens)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cloud(n=5000, seed=0):
    from paper_2302_14801_b200 import PointCloud
    rng = np.random.default_rng(seed)
    return PointCloud(rng.random((n, 3)), rng.integers(0, 256, (n, 3)).astype(np.uint8))


def test_empty_cloud():
    from paper_2302_14801_b200 import BuildConfig, PointCloud, partition
    with pytest.raises(ValueError, match="^cannot partition an empty point cloud$"):
        partition(PointCloud(np.zeros((0, 3)), np.zeros((0, 3), np.uint8)), BuildConfig())


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_coordinates(bad):
    from paper_2302_14801_b200 import BuildConfig, PointCloud, partition
    c = _cloud()
    pos = c.positions.copy()
    pos[1234, 1] = bad
    with pytest.raises(ValueError, match="^point coordinates must be finite$"):
        partition(PointCloud(pos, c.colors), BuildConfig(T=100))


def test_non_finite_fused_entry():
    from paper_2302_14801_b200 import build_lod_points
    c = _cloud()
    pos = c.positions.astype(np.float32)
    pos[7, 2] = np.nan
    with pytest.raises(ValueError, match="^point coordinates must be finite$"):
        build_lod_points(pos, c.colors, T=100)


@pytest.mark.parametrize("kw,msg", [(dict(T=0), "T must be >= 1"),
                                    (dict(max_depth=7), "max_depth must be >= initial_depth"),
                                    (dict(max_depth=17), "max_depth must be <= 16")])
def test_bad_config(kw, msg):
    from paper_2302_14801_b200 import BuildConfig
    with pytest.raises(ValueError, match=f"^{msg}$"):
        BuildConfig(**kw)


def test_unknown_strategy():
    from paper_2302_14801_b200 import BuildConfig, build_lod, partition
    tree = partition(_cloud(), BuildConfig(T=500))
    with pytest.raises(ValueError, match="^unknown sampling strategy: nearest$"):
        build_lod(tree, "nearest", 0)
    # the tree is still usable afterwards
    build_lod(tree, "average", 0)


def test_length_mismatch():
    from paper_2302_14801_b200 import PointCloud
    with pytest.raises(ValueError, match="^positions/colors length mismatch$"):
        PointCloud(np.zeros((3, 3)), np.zeros((2, 3), np.uint8))


@pytest.mark.parametrize("where", ["below", "above"])
def test_point_outside_forced_bounds(where):
    from paper_2302_14801_b200 import AABB, BuildConfig, ConsistencyError, PointCloud
    from paper_2302_14801_b200.partition import Partitioner
    c = _cloud()
    pos = c.positions.copy()
    pos[4321] = (-0.25, 0.5, 0.5) if where == "below" else (0.5, 1.0 + 2.0 ** -20, 0.5)
    with pytest.raises(ConsistencyError, match="^point outside bounds during grid projection$"):
        Partitioner(PointCloud(pos, c.colors), BuildConfig(T=200), bounds=AABB((0.0, 0.0, 0.0), 1.0)).run()


def test_forced_bounds_max_face_is_inside():
    """A point exactly on the forced cube's max face is inside (clipped to the last cell,
    model.py:93-97); the tree matches the oracle's."""
    from oracle import lod_oracle as O
    from paper_2302_14801_b200 import AABB, BuildConfig, PointCloud
    from paper_2302_14801_b200.partition import Partitioner
    c = _cloud(20_000, seed=3)
    pos = c.positions.copy() * 0.5 + 0.25
    pos[:50] = (1.0, 1.0, 1.0)
    tree = Partitioner(PointCloud(pos, c.colors), BuildConfig(T=300), bounds=AABB((0.0, 0.0, 0.0), 1.0)).run()
    sp = O.split(pos, T=300, bounds=((0.0, 0.0, 0.0), 1.0))
    got = {nd.path: nd.point_count for nd in tree.leaves()}
    exp = {p: nd.count for p, nd in sp.nodes.items() if nd.kind == "leaf"}
    assert got == exp


def test_exception_classes_are_the_reference_names():
    from paper_2302_14801_b200 import errors
    assert errors.ConsistencyError.__name__ == "ConsistencyError"
    assert issubclass(errors.ConsistencyError, Exception)
    assert errors.FormatError.__name__ == "FormatError"


def test_stale_tree_on_reused_handle_raises():
    """Trees share a DeviceTree's buffers; a later build on the handle makes an earlier,
    unmaterialised tree refuse access instead of showing the new data."""
    from paper_2302_14801_b200 import BuildConfig, partition
    from paper_2302_14801_b200.device import DeviceTree
    from paper_2302_14801_b200.partition import Partitioner
    dev = DeviceTree()
    a = Partitioner(_cloud(4000, 1), BuildConfig(T=300), device_tree=dev).run()
    kept = Partitioner(_cloud(3000, 2), BuildConfig(T=300), device_tree=dev).run()
    kept_nodes = kept.node_count
    _ = kept.root   # materialised trees stay valid
    Partitioner(_cloud(5000, 3), BuildConfig(T=300), device_tree=dev).run()
    with pytest.raises(RuntimeError, match="reused by a later build"):
        a.root
    assert kept.node_count == kept_nodes and kept.root is not None
    assert partition(_cloud(100, 4), BuildConfig(T=300)).node_count == 1


def test_fused_entry_config_records_what_was_built():
    from paper_2302_14801_b200 import BuildConfig, build_lod_points
    c = _cloud(6000, 5)
    tree = build_lod_points(c.positions, c.colors, mode="random", seed=9, config=BuildConfig(T=700))
    assert tree.config.strategy == "random" and tree.config.seed == 9 and tree.config.T == 700
    with pytest.raises(ValueError, match="conflicts with config.T"):
        build_lod_points(c.positions, c.colors, T=123, config=BuildConfig(T=700))


def test_average_exact_fallback_tiny_arena_retry():
    """LODB200_TINY_ARENA=1 starts every voxelize from a 4096-voxel arena, so the grow-and-retry
    path runs (and, with 70k coincident samples, the u64 exact-sum fallback after it); the
    result must still equal the oracle's."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, sys
sys.path.insert(0, "tests")
from test_gpu_edge import _cloud, _compare
pos, col = _cloud(70_000, 30_000)
_compare(pos, col, 1000, "average")
pos, col = _cloud(2_000, 60_000, seed=5)
_compare(pos, col, 700, "first-come")
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LODB200_TINY_ARENA="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
