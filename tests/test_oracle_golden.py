"""Pin the CPU oracle against digests produced by the real reference.

`tests/golden/*.json.gz` come from `tests/golden/make_golden.py`, which runs the
unmodified `lodforge` partition + build_lod.  Passing here means the oracle's
split (node set, counts, oversized flags, fp64 node bounds, leaf contents in
input order) and its random/average voxels are identical to the reference's.
"""
import numpy as np
import pytest

from conftest import golden_available, load_golden
from cases import CASES, make_input

from helpers import compare_weighted
from oracle import lod_oracle as O

QUICK = [c for c in CASES if c["quick"]]
SLOW_CPU = [c for c in CASES if not c["quick"] and c["name"] != "terrain20M"]


def check_case(case):
    g = load_golden(case["name"])
    pos, col = make_input(case)
    pos64 = np.asarray(pos, np.float64)
    sp = O.split(pos64, **case["cfg"])
    assert [v.hex() for v in sp.world[0]] + [sp.world[1].hex()] == g["world"]
    d = O.split_digest(sp, pos64, col)
    assert d == g["split"], case["name"]
    for mode, exp in g["modes"].items():
        strat, _, seed = mode.partition(":")
        if "error" in exp:
            with pytest.raises(O.ConsistencyError, match="20-bit index limit") as ei:
                O.voxelize(sp, pos64, col, strat, int(seed or 0))
            assert str(ei.value) == exp["error"]
        elif strat == "weighted":
            vox = O.voxelize(sp, pos64, col, strat, 0)
            errors, off, _ = compare_weighted({O.path_str(p): v for p, v in vox.items()}, exp)
            assert not errors and off == 0, (case["name"], errors[:4], off)   # the oracle is exact
        else:
            vox = O.voxelize(sp, pos64, col, strat, int(seed or 0))
            assert O.voxel_digest(vox) == exp, (case["name"], mode)


@pytest.mark.parametrize("case", QUICK, ids=[c["name"] for c in QUICK])
def test_oracle_matches_reference(case):
    check_case(case)


@pytest.mark.slow
@pytest.mark.parametrize("case", SLOW_CPU, ids=[c["name"] for c in SLOW_CPU])
def test_oracle_matches_reference_large(case):
    if not golden_available(case["name"]):
        pytest.skip("golden not generated")
    check_case(case)


# --- known-answer tests of the reference's own test suite, restated on the oracle ---

def test_merge_small_group():            # test_partition.py:48-52
    g = np.zeros((2, 2, 2), np.int64)
    g[:] = 1000
    lv = O.merge_levels(g, 50_000)
    assert lv[0].flat[0] == 8000 and (lv[1] == 0).all()


def test_merge_threshold_flags_parent():  # test_partition.py:54-58
    g = np.zeros((2, 2, 2), np.int64)
    g[0, 0, 0], g[1, 0, 0] = 49_999, 1
    lv = O.merge_levels(g, 50_000)
    assert lv[0].flat[0] == O.UNMERGEABLE and lv[1][0, 0, 0] == 49_999 and lv[1][1, 0, 0] == 1


def test_merge_unmergeable_propagates():  # test_partition.py:60-64
    g = np.zeros((2, 2, 2), np.int64)
    g[0, 0, 0], g[1, 1, 1] = O.UNMERGEABLE, 3
    lv = O.merge_levels(g, 50_000)
    assert lv[0].flat[0] == O.UNMERGEABLE and lv[1][1, 1, 1] == 3


def test_merge_cascade():                 # test_partition.py:70-74
    g = np.zeros((4, 4, 4), np.int64)
    g[0, 0, 0], g[3, 3, 3] = 5, 7
    lv = O.merge_levels(g, 100)
    assert lv[0].flat[0] == 12 and (lv[1] == 0).all() and (lv[2] == 0).all()


def test_cell_goldens():                  # test_model.py:48-55
    lo, s = (0.0, 0.0, 0.0), 1.0
    pts = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [0.5, 0.25, 0.75]])
    assert O.grid_cells(pts, lo, s, 256).tolist() == [[0, 0, 0], [255, 255, 255], [128, 64, 192]]
    with pytest.raises(O.ConsistencyError):
        O.grid_cells(np.array([[1.5, 0.5, 0.5]]), lo, s, 256)


def test_node_bounds_goldens():           # test_model.py:17-32
    assert O.node_bounds((0, 0, 0), 2, (7,)) == ((1, 1, 1), 1)
    assert O.node_bounds((4, 4, 4), 8, (1,)) == ((8, 4, 4), 4)


def test_average_rounding():              # test_sampling.py:127-138
    cells = np.array([[5, 5, 5], [5, 5, 5]])
    assert O.extract_average(cells, np.array([[200, 0, 0], [100, 0, 0]], np.uint8))[1][0].tolist() == [150, 0, 0]
    assert O.extract_average(cells, np.array([[200, 0, 0], [101, 0, 0]], np.uint8))[1][0].tolist() == [151, 0, 0]


def test_random_limit():                  # test_sampling.py:119-124
    with pytest.raises(O.ConsistencyError):
        O.extract_random(np.zeros((1 << 20, 3), np.int64), np.zeros((1 << 20, 3), np.uint8), 0, 0)


def test_random_key_encoding():           # test_sampling.py:95-99
    assert (0xFFFFFFFF & 0xFFF00000) | (0x12345 & 0x000FFFFF) == 0xFFF12345
