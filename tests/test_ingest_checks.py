"""Ingest (reference ingest.py:59-221) and structural checks (checks.py:18-92).

CPU: the host readers follow the reference's tests (test_ingest.py TestLas / TestPly) and
error paths.  GPU: files streamed to HBM and decoded by lod_ingest_las / lod_ingest_ply
are bit-identical to the host readers (every LAS point format, PLY property types);
build_file == partition(read_cloud) + build_lod; device run_checks == the host rules on
the materialised tree, including detected violations."""
import struct

import numpy as np
import pytest

from paper_2302_14801_b200 import FormatError, PointCloud
from paper_2302_14801_b200.ingest import read_cloud, read_las, read_ply, write_ply

_RECLEN = {0: 20, 1: 28, 2: 26, 3: 34, 6: 30, 7: 36, 8: 38}
_RGB = {2: 20, 3: 28, 7: 30, 8: 30}


def las_bytes(ints, fmt=0, rgb=None, scale=(0.001,) * 3, offset=(0.0,) * 3, version=(1, 2), pad=0):
    """Minimal LAS file: integer coordinates `ints` (n,3), optional 16-bit colours."""
    reclen = _RECLEN[fmt] + pad
    header = bytearray(227)
    header[0:4] = b"LASF"
    header[24], header[25] = version
    struct.pack_into("<I", header, 96, 227)
    header[104] = fmt
    struct.pack_into("<H", header, 105, reclen)
    struct.pack_into("<I", header, 107, len(ints))
    struct.pack_into("<3d", header, 131, *scale)
    struct.pack_into("<3d", header, 155, *offset)
    rec = np.zeros((len(ints), reclen), np.uint8)
    rec[:, :12] = np.asarray(ints, "<i4").reshape(-1, 3).view(np.uint8).reshape(-1, 12)
    if rgb is not None:
        b = _RGB[fmt]
        rec[:, b:b + 6] = np.asarray(rgb, "<u2").reshape(-1, 3).view(np.uint8).reshape(-1, 6)
    return bytes(header) + rec.tobytes()


class TestHostReaders:
    def test_las_single_point_grey(self, tmp_path):
        f = tmp_path / "a.las"
        f.write_bytes(las_bytes([(1000, 2000, 3000)]))
        c = read_las(f)
        assert np.allclose(c.positions[0], (1, 2, 3)) and tuple(c.colors[0]) == (128, 128, 128)

    def test_las_rgb_high_byte(self, tmp_path):
        f = tmp_path / "a.las"
        f.write_bytes(las_bytes([(0, 0, 0)], fmt=2, rgb=[(65535, 0, 256)]))
        assert tuple(read_las(f).colors[0]) == (255, 0, 1)

    def test_las_errors(self, tmp_path):
        f = tmp_path / "a.las"
        f.write_bytes(b"XXXX" + las_bytes([(0, 0, 0)])[4:])
        with pytest.raises(FormatError):
            read_las(f)
        f.write_bytes(las_bytes([(0, 0, 0), (1, 1, 1)])[:-10])
        with pytest.raises(IOError):
            read_las(f)
        f.write_bytes(las_bytes([])[:100])
        with pytest.raises(FormatError, match="truncated"):
            read_las(f)
        b = bytearray(las_bytes([(0, 0, 0)]))
        b[104] = 0x80
        f.write_bytes(bytes(b))
        with pytest.raises(FormatError, match="LAZ"):
            read_las(f)
        assert len(read_las(_write(tmp_path, las_bytes([])))) == 0

    def test_ply_ascii_and_grey(self, tmp_path):
        f = tmp_path / "a.ply"
        f.write_text("ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nproperty float y\n"
                     "property float z\nproperty uchar red\nproperty uchar green\nproperty uchar blue\n"
                     "end_header\n0 0 0 255 0 0\n")
        c = read_ply(f)
        assert tuple(c.colors[0]) == (255, 0, 0)
        f.write_text("ply\nformat ascii 1.0\nelement vertex 1\nproperty double x\nproperty double y\n"
                     "property double z\nend_header\n0.5 0.25 0.125\n")
        assert tuple(read_ply(f).colors[0]) == (128, 128, 128)

    def test_ply_errors(self, tmp_path):
        f = tmp_path / "a.ply"
        for body, err in [("format binary_big_endian 1.0\nelement vertex 0\nproperty float x\nproperty float y\n"
                           "property float z\n", "big-endian"),
                          ("format ascii 1.0\nelement vertex 1\nproperty float x\nproperty float y\n", "x/y/z"),
                          ("format ascii 1.0\nelement face 1\nproperty float x\n", "vertex element")]:
            f.write_text("ply\n" + body + "end_header\n0 0\n")
            with pytest.raises(FormatError, match=err):
                read_ply(f)

    def test_ply_binary_round_trip(self, tmp_path):
        rng = np.random.default_rng(3)
        cloud = PointCloud(rng.random((500, 3)), rng.integers(0, 256, (500, 3)).astype(np.uint8))
        f = tmp_path / "a.ply"
        write_ply(f, cloud)
        back = read_cloud(f)
        assert np.array_equal(back.positions, cloud.positions) and np.array_equal(back.colors, cloud.colors)


def _write(tmp_path, data, name="z.las"):
    p = tmp_path / name
    p.write_bytes(data)
    return p


def _ply_binary(path, props, cols):
    """binary_little_endian PLY with the given (name, ply type, numpy type) properties."""
    n = len(cols[props[0][0]])
    head = f"ply\nformat binary_little_endian 1.0\nelement vertex {n}\n"
    head += "".join(f"property {t} {name}\n" for name, t, _ in props) + "end_header\n"
    rec = np.zeros(n, [(name, dt) for name, _, dt in props])
    for name, _, _ in props:
        rec[name] = cols[name]
    path.write_bytes(head.encode() + rec.tobytes())


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", sorted(_RECLEN))
def test_device_las_decode_matches_host(tmp_path, fmt):
    from paper_2302_14801_b200.device import unpack_records
    from paper_2302_14801_b200.ingest import load_points
    rng = np.random.default_rng(fmt)
    n = 70_001
    ints = rng.integers(-2**31, 2**31 - 1, (n, 3))
    rgb = rng.integers(0, 65536, (n, 3)) if fmt in _RGB else None
    f = _write(tmp_path, las_bytes(ints, fmt, rgb, scale=(1e-3, 3.3e-4, 0.01), offset=(1e5, -7.5, 3.25),
                                   version=(1, 4) if fmt >= 6 else (1, 2), pad=3), "p.las")
    host = read_las(f)
    dp = load_points(f, chunk_bytes=1 << 20)   # several double-buffered chunks
    pos, col = unpack_records(dp.records.cpu().numpy()[: n * 32], dp.fmt)
    assert np.array_equal(pos.view(np.uint64), host.positions.view(np.uint64))
    assert np.array_equal(col, host.colors)


@pytest.mark.gpu
@pytest.mark.parametrize("ptypes", [("float", "uchar"), ("double", "ushort"), ("int", "float"), ("short", "uint"),
                                    ("uint", "double"), ("double", None)])
def test_device_ply_decode_matches_host(tmp_path, ptypes):
    from paper_2302_14801_b200.device import unpack_records
    from paper_2302_14801_b200.ingest import _PLY_SCALARS, load_points
    rng = np.random.default_rng(7)
    n = 50_003
    pt, ct = ptypes
    cols = {}
    props = [("nx", "float", "<f4")]
    cols["nx"] = rng.random(n).astype(np.float32)
    for a in "xyz":
        dt = np.dtype(_PLY_SCALARS[pt])
        cols[a] = (rng.random(n) * 1000 - 500).astype(dt) if dt.kind == "f" else rng.integers(
            np.iinfo(dt).min, np.iinfo(dt).max, n, dtype=dt)
        props.append((a, pt, _PLY_SCALARS[pt]))
    if ct:
        for c in ("red", "green", "blue"):
            dt = np.dtype(_PLY_SCALARS[ct])
            cols[c] = (rng.random(n) * 255).astype(dt) if dt.kind == "f" else rng.integers(0, min(
                np.iinfo(dt).max, 4000), n, dtype=dt)
            props.append((c, ct, _PLY_SCALARS[ct]))
    f = tmp_path / "p.ply"
    _ply_binary(f, props, cols)
    host = read_ply(f)
    dp = load_points(f, chunk_bytes=1 << 20)
    rs = 16 if dp.fmt == 0 else 32
    pos, col = unpack_records(dp.records.cpu().numpy()[: n * rs], dp.fmt)
    assert np.array_equal(pos, host.positions)
    assert np.array_equal(col, host.colors)


@pytest.mark.gpu
def test_build_file_matches_host_path(tmp_path):
    """build_file (device ingest) == partition(read_cloud(file)) + build_lod, node by node."""
    from helpers import tree_split_digest, tree_voxel_digest
    from paper_2302_14801_b200 import BuildConfig, build_lod, partition
    from paper_2302_14801_b200.generators import reference_cloud
    from paper_2302_14801_b200.ingest import build_file
    c = reference_cloud("stadium", 150_000, 4)
    f = tmp_path / "s.ply"
    write_ply(f, PointCloud(c.positions, c.colors))
    cfg = BuildConfig(T=3000)
    a = build_file(f, cfg, "average", 0)
    b = partition(read_cloud(f), cfg)
    build_lod(b, "average", 0)
    assert tree_split_digest(a) == tree_split_digest(b)
    assert tree_voxel_digest(a) == tree_voxel_digest(b)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["first-come", "average", None])
def test_device_checks_match_host_rules(strategy):
    from paper_2302_14801_b200 import BuildConfig, Octree, build_lod, partition
    from paper_2302_14801_b200.checks import all_passed, run_checks
    from paper_2302_14801_b200.generators import reference_cloud
    c = reference_cloud("two-scans", 120_000, 2)
    tree = partition(PointCloud(c.positions, c.colors), BuildConfig(T=2000))
    if strategy:
        build_lod(tree, strategy, 0)
    dev = run_checks(tree, expected_points=120_000)
    host = run_checks(Octree(tree.root, tree.world_bounds, tree.config), expected_points=120_000)
    assert [(r.name, r.passed, r.detail) for r in dev] == [(r.name, r.passed, r.detail) for r in host]
    assert all_passed(dev) == (strategy is not None)
    bad = run_checks(tree, expected_points=5)
    assert not bad[0].passed and bad[0].detail == "leaf points 120000, expected 5"
    tight = run_checks(tree.__class__(tree.device_tree, BuildConfig(T=10)), expected_points=120_000)
    assert not next(r for r in tight if r.name == "capacity").passed


# ---------------------------------------------------------------------------
# pinned to the REAL reference: tests/golden/ingest_checks.json.gz (make_ingest_golden.py ran
# lodforge.ingest.read_las / read_ply and lodforge.checks.run_checks on these inputs)
# ---------------------------------------------------------------------------

def _ingest_golden():
    from conftest import load_golden
    return load_golden("ingest_checks")


def _golden_files(tmp_path):
    import ingest_cases as IC
    out = []
    for name, data in IC.files().items():
        p = tmp_path / name
        p.write_bytes(data)
        out.append((name, p))
    return out


def _sha(a):
    import hashlib
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_host_readers_match_reference_goldens(tmp_path):
    g = _ingest_golden()["files"]
    for name, p in _golden_files(tmp_path):
        c = read_cloud(p)
        assert [len(c), _sha(c.positions), _sha(c.colors)] == g[name][:3], name


@pytest.mark.gpu
def test_device_decode_matches_reference_goldens(tmp_path):
    """lod_ingest_las / lod_ingest_ply (via load_points, streamed in double-buffered chunks)
    decode to exactly the reference's read_las / read_ply arrays (sha1 of f64 positions and
    u8 colours), for every LAS point format, LAS 1.4 64-bit counts, binary PLY property types
    and ASCII PLY."""
    from paper_2302_14801_b200.device import unpack_records
    from paper_2302_14801_b200.ingest import load_points
    g = _ingest_golden()["files"]
    for name, p in _golden_files(tmp_path):
        dp = load_points(p, chunk_bytes=1 << 18)
        n = g[name][0]
        rs = 16 if dp.fmt == 0 else 32
        pos, col = unpack_records(dp.records.cpu().numpy()[: n * rs], dp.fmt)
        assert [n, _sha(pos), _sha(col)] == g[name][:3], name


@pytest.mark.gpu
def test_device_checks_match_reference_goldens():
    """Device run_checks (lod_tree_checks) == the reference's run_checks on the same trees:
    names, pass/fail and detail text (first offending paths in DFS order)."""
    import ingest_cases as IC
    from paper_2302_14801_b200 import BuildConfig, build_lod, partition
    from paper_2302_14801_b200.checks import run_checks
    from paper_2302_14801_b200.generators import reference_cloud
    gold = _ingest_golden()["checks"]
    for kind, n, seed, T in IC.CHECK_CASES:
        exp = gold[f"{kind}_{n}_{seed}_T{T}"]
        c = reference_cloud(kind, n, seed)
        tree = partition(PointCloud(c.positions, c.colors), BuildConfig(T=T))

        def rec(r):
            return [[x.name, bool(x.passed), x.detail] for x in r]

        assert rec(run_checks(tree, expected_points=n)) == exp["split"]
        build_lod(tree, "first-come", 0)
        assert rec(run_checks(tree, expected_points=n)) == exp["first-come"]
        build_lod(tree, "average", 0)
        assert rec(run_checks(tree, expected_points=n)) == exp["average"]
        assert rec(run_checks(tree, expected_points=5)) == exp["expected5"]
        tight = tree.__class__(tree.device_tree, BuildConfig(T=10))
        tight._generation = tree._generation
        assert rec(run_checks(tight, expected_points=n)) == exp["tightT10"]
