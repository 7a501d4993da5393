"""VLPC codec (reference codec.py): byte-identical files from the device encoder.

CPU tests cover the host side (path ordering, header parsing, FormatError paths, the
host encoder round trip).  GPU tests encode trees built on the B200 and compare length +
SHA-1 with the files the reference itself wrote for the same inputs
(`tests/golden/*.json.gz` "vlpc", made by make_golden.py), then check decode -> encode
identity (test_acceptance.py:260-276)."""
import hashlib
import io
import itertools
import random

import numpy as np
import pytest

from conftest import load_golden
from cases import CASES, make_input


def test_path_sort_keys_match_tuple_order():
    from paper_2302_14801_b200.codec import path_sort_keys
    rng = random.Random(5)
    paths = {()}
    for _ in range(400):
        d = rng.randint(1, 16)
        p = tuple(rng.randint(0, 7) for _ in range(d))
        for k in range(d + 1):
            paths.add(p[:k])
    paths = sorted(paths, key=len)
    cells = np.zeros((len(paths), 3), np.uint16)
    depth = np.array([len(p) for p in paths], np.uint8)
    for i, p in enumerate(paths):
        for o in p:
            cells[i, 0] = (cells[i, 0] << 1) | (o & 1)
            cells[i, 1] = (cells[i, 1] << 1) | ((o >> 1) & 1)
            cells[i, 2] = (cells[i, 2] << 1) | (o >> 2)
    order = np.argsort(path_sort_keys(cells, depth), kind="stable")
    assert [paths[i] for i in order] == sorted(paths)


def test_header_errors():
    from paper_2302_14801_b200 import FormatError
    from paper_2302_14801_b200.codec import _HEADER, decode, read_header
    with pytest.raises(FormatError, match="too small"):
        read_header(b"VLPC")
    bad = bytearray(_HEADER.pack(b"VLPX", 1, 0, 0, 0, 1, 10, 0, 0, 0, 0))
    with pytest.raises(FormatError, match="bad magic"):
        read_header(bytes(bad))
    with pytest.raises(FormatError, match="unsupported VLPC version 2"):
        read_header(_HEADER.pack(b"VLPC", 2, 0, 0, 0, 1, 10, 0, 0, 0, 0))
    with pytest.raises(FormatError, match="truncated node table"):
        decode(io.BytesIO(_HEADER.pack(b"VLPC", 1, 0, 0, 0, 1, 10, 0, 1, 0, 0)))
    with pytest.raises(FormatError, match="missing root node"):
        decode(io.BytesIO(_HEADER.pack(b"VLPC", 1, 0, 0, 0, 1, 10, 0, 0, 0, 0)))


def test_host_encoder_roundtrip():
    """decode(encode(t)) re-encodes to the same bytes (host objects only)."""
    from paper_2302_14801_b200 import AABB, BuildConfig, Octree, OctreeNode
    from paper_2302_14801_b200.codec import decode, encode_bytes
    from paper_2302_14801_b200.model import bounds_at
    world = AABB((0.0, 0.0, 0.0), 1.0)
    rng = np.random.default_rng(0)
    root = OctreeNode((), world, children=[None] * 8)
    root.voxel_coords = rng.integers(0, 128, (5, 3)).astype(np.uint8)
    root.voxel_colors = rng.integers(0, 256, (5, 3)).astype(np.uint8)
    for o in (1, 6):
        b = bounds_at(world, (o,))
        pts = b.min_array() + rng.random((7, 3)) * b.size
        root.children[o] = OctreeNode((o,), b, None, pts.astype(np.float32).astype(np.float64),
                                      rng.integers(0, 256, (7, 3)).astype(np.uint8))
    tree = Octree(root, world, BuildConfig(T=10, strategy="average", seed=4))
    blob = encode_bytes(tree)
    again = encode_bytes(decode(io.BytesIO(blob)))
    assert again == blob


QUICK = [c for c in CASES if c["quick"]]


@pytest.mark.gpu
@pytest.mark.parametrize("case", QUICK, ids=[c["name"] for c in QUICK])
def test_device_encode_matches_reference_file(case):
    from paper_2302_14801_b200 import BuildConfig, PointCloud, build_lod, partition
    from paper_2302_14801_b200.codec import decode, encode, encode_bytes
    g = load_golden(case["name"])
    pos, col = make_input(case)
    tree = partition(PointCloud(np.asarray(pos, np.float64), col), BuildConfig(**case["cfg"]))
    assert g.get("vlpc"), "golden lacks VLPC digests"
    for mode, (length, digest) in g["vlpc"].items():
        strat, _, seed = mode.partition(":")
        build_lod(tree, strat, int(seed or 0))
        tree.config.strategy, tree.config.seed = strat, int(seed or 0)
        buf = io.BytesIO()
        n = encode(tree, buf)
        blob = buf.getvalue()
        assert n == len(blob) == length, (case["name"], mode)
        assert hashlib.sha1(blob).hexdigest() == digest, (case["name"], mode)
        assert encode_bytes(decode(io.BytesIO(blob))) == blob   # codec identity (test_acceptance.py:270-275)
