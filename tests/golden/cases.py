"""Golden-case registry shared by `make_golden.py` (runs the real reference, in the
build container only) and the tests (run anywhere, regenerate the same inputs
from `paper_2302_14801_b200.generators`).

A case is (name, input spec, BuildConfig kwargs, sampling modes).
Input spec kinds:
  ("ref", kind, n, seed)           reference preset (ingest.py:229-271), float64 coords
  ("syn", kind, n, seed)           BASELINE synthetic config, float32 coords
  ("tile", (x, y, z), n)           n copies of one point
  ("maxface", k)                   [[0,0,0],[1,1,1]] * k
  ("literal", name)                explicit points stored in the fixture
Optional color override: ("const", (r, g, b)).
Modes: "average" or "random:<seed>".
"""
from __future__ import annotations

import random as _pyrandom

import numpy as np

from paper_2302_14801_b200.generators import reference_cloud, synthetic_cloud


def _acceptance03_cases():
    """test_acceptance.py:97-107 draws 19 cases from random.Random(2024) after a fixed first case."""
    draw = _pyrandom.Random(2024)
    kinds = ["uniform-cube", "stadium", "two-scans", "checker-plane"]
    out = [("uniform-cube", 100_000, 0, 5000)]
    while len(out) < 20:
        out.append((draw.choice(kinds), draw.randint(2_000, 100_000), draw.randint(0, 10_000),
                    draw.choice([500, 1000, 2000, 5000])))
    return out


CASES = []


def _add(name, spec, cfg, modes, color=None, quick=True, weighted=False):
    """Every case also records the reference's "first-come" output (the reference default,
    model.py:115); `weighted` cases also store the reference's "weighted" colours in full
    (compared within +-1 per channel, SPEC.md "Weighted accumulation order")."""
    modes = list(modes) + ["first-come"] + (["weighted"] if weighted else [])
    CASES.append(dict(name=name, spec=spec, cfg=cfg, modes=modes, color=color, quick=quick))


# test_partition.py:146-162 oracle-equivalence cases (+ sampling on the same trees)
for kind, n, seed, T in [("uniform-cube", 20_000, 1, 1000), ("uniform-cube", 5_000, 2, 300),
                         ("stadium", 30_000, 3, 1500), ("two-scans", 20_000, 4, 2000),
                         ("checker-plane", 10_000, 5, 800)]:
    _add(f"part_{kind}_{n}_{seed}_T{T}", ("ref", kind, n, seed), dict(T=T), ["average", "random:11"], weighted=True)

# test_acceptance.py:97-120 randomized partition cases
for kind, n, seed, T in _acceptance03_cases():
    _add(f"acc03_{kind}_{n}_{seed}_T{T}", ("ref", kind, n, seed), dict(T=T), ["average", "random:3"])

# test_acceptance.py:123-151 sampling datasets (T=1500)
for kind, n, seed in [("uniform-cube", 60_000, 6), ("uniform-cube", 40_000, 7),
                      ("two-scans", 40_000, 8), ("stadium", 50_000, 9)]:
    _add(f"acc04_{kind}_{n}_{seed}", ("ref", kind, n, seed), dict(T=1500), ["average", "random:3"], weighted=True)

# test_sampling.py small_tree fixtures
_add("small_tree_30k", ("ref", "uniform-cube", 30_000, 1), dict(T=2000), ["average", "random:9", "random:5"])
_add("small_tree_25k", ("ref", "uniform-cube", 25_000, 1), dict(T=1500), ["average", "random:11"], weighted=True)
_add("const_color_20k", ("ref", "uniform-cube", 20_000, 3), dict(T=1000), ["average", "random:2"],
     color=(12, 200, 99), weighted=True)

# structural edge cases (test_partition.py:107-136, test_sampling.py:224-232)
_add("single_point", ("literal", "single"), dict(), ["average", "random:0"], weighted=True)
_add("identical_2000_T500", ("tile", (0.25, 0.5, 0.75), 2000), dict(T=500), ["average", "random:0"], weighted=True)
_add("maxface_600", ("maxface", 600), dict(T=1000), ["average", "random:0"], weighted=True)
_add("sparse_cluster_T50", ("literal", "sparse200"), dict(T=50), ["average", "random:1"], weighted=True)
_add("uniform_40k_single_leaf", ("ref", "uniform-cube", 40_000, 42), dict(), ["average"])
_add("uniform_100k_T50k", ("ref", "uniform-cube", 100_000, 42), dict(), ["average", "random:0"])
_add("uniform_300k_T20k", ("ref", "uniform-cube", 300_000, 42), dict(T=20_000), ["average", "random:0"])
_add("stadium_600k_s7", ("ref", "stadium", 600_000, 7), dict(), ["average", "random:0"], quick=False)
_add("const_color_100k", ("ref", "uniform-cube", 100_000, 4), dict(), ["average", "random:1"],
     color=(31, 177, 92))
_add("depth_limit_md10", ("ref", "stadium", 200_000, 5), dict(T=2000, max_depth=10), ["average"])
_add("initial6_ext3", ("ref", "stadium", 200_000, 6), dict(T=3000, initial_depth=6, extension_depth=3),
     ["average", "random:4"])

# test_acceptance.py:52-68 module fixture builds (default config)
_add("acc_uniform_1M", ("ref", "uniform-cube", 1_000_000, 1), dict(), ["average", "random:0"], quick=False)
_add("acc_stadium_1M", ("ref", "stadium", 1_000_000, 1), dict(), ["average", "random:0"], quick=False)
_add("stadium_2M_random_limit", ("ref", "stadium", 2_000_000, 1), dict(), ["random:0", "average"],
     quick=False)
_add("acc_plane_100k", ("ref", "checker-plane", 100_000, 1), dict(), ["average", "random:0"])
_add("acc_twoscans_200k", ("ref", "two-scans", 200_000, 1), dict(), ["average", "random:11"])
# > 2^11 leaves: the two-pass distribute and thousands of leaf parents
_add("many_leaves_400k_T100", ("ref", "uniform-cube", 400_000, 3), dict(T=100), ["average", "random:5"],
     quick=False)
_add("many_leaves_stadium_300k_T60", ("ref", "stadium", 300_000, 8), dict(T=60), ["average"], quick=False)

# BASELINE configs; float32 coordinates
_add("sphere1M", ("syn", "sphere", 1_000_000, 1), dict(), ["random:0", "average"], quick=False)
_add("terrain2M", ("syn", "terrain", 2_000_000, 2), dict(), ["average", "random:0"], quick=False)
_add("terrain20M", ("syn", "terrain", 20_000_000, 2), dict(), ["average", "random:0"], quick=False)
_add("cluster1500k_T2000", ("syn", "cluster", 1_500_000, 4), dict(T=2000), ["average", "random:0"],
     quick=False)
_add("scene2M", ("syn", "scene", 2_000_000, 3), dict(), ["average", "random:0"], quick=False)
_add("surface1M", ("syn", "surface", 1_000_000, 5), dict(), ["average", "random:0"], quick=False)


def literal_points(name):
    if name == "single":
        return np.array([[0.3, 0.4, 0.5]]), np.array([[1, 2, 3]], np.uint8)
    if name == "sparse200":   # test_partition.py:97-104
        g = np.random.default_rng(0)
        pos = g.random((200, 3)) * 0.001
        pos[0] = (0.9, 0.9, 0.9)
        return pos, np.zeros((200, 3), np.uint8)
    raise KeyError(name)


def make_input(case):
    """(positions, colors) for a case; positions float64 (ref/literal) or float32 (syn)."""
    spec = case["spec"]
    if spec[0] == "ref":
        c = reference_cloud(spec[1], spec[2], spec[3])
        pos, col = c.positions, c.colors
    elif spec[0] == "syn":
        pos, col = synthetic_cloud(spec[1], spec[2], spec[3])
    elif spec[0] == "tile":
        pos = np.tile(np.array([spec[1]], np.float64), (spec[2], 1))
        col = np.zeros((spec[2], 3), np.uint8)
    elif spec[0] == "maxface":
        pos = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]] * spec[1])
        col = np.zeros((len(pos), 3), np.uint8)
    elif spec[0] == "literal":
        pos, col = literal_points(spec[1])
    else:
        raise ValueError(spec)
    if case.get("color") is not None:
        col = np.empty_like(col)
        col[:] = case["color"]
    return pos, col


def by_name(name):
    for c in CASES:
        if c["name"] == name:
            return c
    raise KeyError(name)
