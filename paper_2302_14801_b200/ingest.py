"""File ingest for the B200 path (reference ingest.py:59-221).

Host readers with the reference's signatures and semantics (`read_las`, `read_ply`,
`write_ply`, `read_cloud`), and the device path the construction uses for files:

    load_points(path) -> DevicePoints      # record bytes streamed to HBM, decoded there
    build_file(path, config, strategy, seed) -> GpuOctree

`load_points` parses only the header on the host.  The point-record region of the file is
read in chunks into two pinned staging buffers and copied to HBM asynchronously (the
disk read of chunk k+1 overlaps the PCIe copy of chunk k); `lod_ingest_las` /
`lod_ingest_ply` then decode every record on the device (LAS: X*scale+offset in fp64 and
16-bit colour >> 8; PLY: any scalar type widened to f64, colours cast to u8).  ASCII PLY is
parsed on the host (text) and uploaded.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _abi
from .errors import FormatError
from .model import PointCloud

# --------------------------------------------------------------------------- LAS
_LAS_MIN_RECLEN = {0: 20, 1: 28, 2: 26, 3: 34, 6: 30, 7: 36, 8: 38}   # ingest.py:55
_LAS_RGB_OFFSET = {2: 20, 3: 28, 7: 30, 8: 30}                        # ingest.py:56


@dataclass
class LasHeader:
    n: int
    fmt: int
    reclen: int
    offset_to_points: int
    scale: tuple
    offset: tuple

    @property
    def rgb_offset(self) -> int:
        return _LAS_RGB_OFFSET.get(self.fmt, -1)


def las_header(f) -> LasHeader:
    """Header of an LAS 1.2-1.4 file (ingest.py:61-88), same errors."""
    header = f.read(227)
    if len(header) < 227:
        raise FormatError("LAS header truncated")
    if header[:4] != b"LASF":
        raise FormatError("not an LAS file (missing LASF magic)")
    ver = (header[24], header[25])
    offset_to_points = struct.unpack_from("<I", header, 96)[0]
    fmt_byte = header[104]
    if fmt_byte & 0x80:
        raise FormatError("compressed LAS (LAZ) is not supported")
    fmt = fmt_byte & 0x3F
    reclen = struct.unpack_from("<H", header, 105)[0]
    n = struct.unpack_from("<I", header, 107)[0]
    scale = struct.unpack_from("<3d", header, 131)
    offset = struct.unpack_from("<3d", header, 155)
    if ver >= (1, 4):
        full = header + f.read(375 - 227)
        if len(full) >= 255:
            n64 = struct.unpack_from("<Q", full, 247)[0]
            if n64:
                n = n64
    if fmt not in _LAS_MIN_RECLEN:
        raise FormatError(f"unsupported LAS point format {fmt}")
    if reclen < _LAS_MIN_RECLEN[fmt]:
        raise FormatError(f"record length {reclen} too short for format {fmt}")
    return LasHeader(n, fmt, reclen, offset_to_points, scale, offset)


def read_las(path) -> PointCloud:
    """Read an LAS 1.2-1.4 file (point formats 0-3 and 6-8, uncompressed) -- ingest.py:59-116."""
    with open(path, "rb") as f:
        h = las_header(f)
        if h.n == 0:
            return PointCloud(np.empty((0, 3)), np.empty((0, 3), np.uint8))
        f.seek(h.offset_to_points)
        raw = f.read(h.n * h.reclen)
        if len(raw) < h.n * h.reclen:
            raise IOError("truncated LAS point records")
    names, formats, offsets = ["x", "y", "z"], ["<i4"] * 3, [0, 4, 8]
    if h.rgb_offset >= 0:
        names += ["red", "green", "blue"]
        formats += ["<u2"] * 3
        offsets += [h.rgb_offset, h.rgb_offset + 2, h.rgb_offset + 4]
    rec = np.frombuffer(raw, np.dtype({"names": names, "formats": formats, "offsets": offsets,
                                       "itemsize": h.reclen}), count=h.n)
    pos = np.empty((h.n, 3))
    for i, (axis, sc, off) in enumerate(zip("xyz", h.scale, h.offset)):
        pos[:, i] = rec[axis].astype(np.float64) * sc + off
    if h.rgb_offset >= 0:
        col = np.stack([(rec[c] >> 8).astype(np.uint8) for c in ("red", "green", "blue")], axis=1)
    else:
        col = np.full((h.n, 3), 128, np.uint8)
    return PointCloud(pos, col)


# --------------------------------------------------------------------------- PLY
_PLY_SCALARS = {                                                      # ingest.py:122-131
    "char": "i1", "int8": "i1", "uchar": "u1", "uint8": "u1", "short": "<i2", "int16": "<i2",
    "ushort": "<u2", "uint16": "<u2", "int": "<i4", "int32": "<i4", "uint": "<u4", "uint32": "<u4",
    "float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8",
}
_PLY_CODES = {"i1": 0, "u1": 1, "<i2": 2, "<u2": 3, "<i4": 4, "<u4": 5, "<f4": 6, "<f8": 7}  # lod_ply_type


@dataclass
class PlyHeader:
    fmt: str
    count: int
    props: list
    body_start: int


def ply_header(data: bytes) -> PlyHeader:
    """Header of an ascii / binary-little-endian PLY (ingest.py:137-170), same errors."""
    end = data.find(b"end_header")
    if not data.startswith(b"ply") or end < 0:
        raise FormatError("not a PLY file")
    body_start = data.find(b"\n", end) + 1
    fmt, elements = None, []
    for line in data[:end].decode("ascii", errors="replace").splitlines():
        tok = line.split()
        if not tok:
            continue
        if tok[0] == "format":
            fmt = tok[1]
        elif tok[0] == "element":
            elements.append((tok[1], int(tok[2]), []))
        elif tok[0] == "property":
            if not elements:
                raise FormatError("PLY property before any element")
            elements[-1][2].append((tok[-1], "list" if tok[1] == "list" else tok[1]))
    if fmt == "binary_big_endian":
        raise FormatError("big-endian PLY is not supported")
    if fmt not in ("ascii", "binary_little_endian"):
        raise FormatError(f"unsupported PLY format: {fmt}")
    if not elements or elements[0][0] != "vertex":
        raise FormatError("PLY vertex element must come first")
    _, count, props = elements[0]
    if any(p[1] == "list" for p in props):
        raise FormatError("list properties on vertices are not supported")
    if not {"x", "y", "z"} <= {p[0] for p in props}:
        raise FormatError("PLY vertex element lacks x/y/z properties")
    return PlyHeader(fmt, count, props, body_start)


def _ply_dtype(props) -> np.dtype:
    try:
        return np.dtype([(name, _PLY_SCALARS[typ]) for name, typ in props])
    except KeyError as e:
        raise FormatError(f"unsupported PLY property type: {e}")


def _ply_columns(data: bytes, h: PlyHeader):
    names = [p[0] for p in h.props]
    if h.fmt == "ascii":
        rows = data[h.body_start:].decode("ascii").split()
        ncols = len(h.props)
        vals = (np.array(rows[: h.count * ncols], dtype=np.float64).reshape(h.count, ncols) if h.count > 0
                else np.empty((0, ncols)))
        cols = {name: vals[:, i] for i, (name, _) in enumerate(h.props)}
    else:
        dt = _ply_dtype(h.props)
        if len(data) - h.body_start < h.count * dt.itemsize:
            raise IOError("truncated PLY vertex data")
        rec = np.frombuffer(data, dtype=dt, count=h.count, offset=h.body_start)
        cols = {name: rec[name] for name, _ in h.props}
    pos = np.stack([cols["x"], cols["y"], cols["z"]], axis=1).astype(np.float64)
    if {"red", "green", "blue"} <= set(names):
        col = np.stack([cols["red"], cols["green"], cols["blue"]], axis=1).astype(np.uint8)
    else:
        col = np.full((h.count, 3), 128, np.uint8)
    return pos, col


def read_ply(path) -> PointCloud:
    """Read an ascii or binary-little-endian PLY with x,y,z and optional red,green,blue -- ingest.py:134-198."""
    with open(path, "rb") as f:
        data = f.read()
    return PointCloud(*_ply_columns(data, ply_header(data)))


def write_ply(path, cloud: PointCloud) -> None:
    """Binary-little-endian PLY with float64 positions and uint8 colours -- ingest.py:201-221."""
    n = len(cloud)
    header = ("ply\nformat binary_little_endian 1.0\n"
              f"element vertex {n}\n"
              "property double x\nproperty double y\nproperty double z\n"
              "property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n")
    rec = np.empty(n, dtype=[("pos", "<f8", 3), ("rgb", "u1", 3)])
    rec["pos"] = cloud.positions
    rec["rgb"] = cloud.colors
    with open(path, "wb") as f:
        f.write(header.encode("ascii"))
        f.write(rec.tobytes())


def read_cloud(path) -> PointCloud:
    """`.las` -> read_las, anything else -> read_ply (cli.py:60-64)."""
    return read_las(path) if str(path).lower().endswith(".las") else read_ply(path)


# --------------------------------------------------------------------------- device path
@dataclass
class DevicePoints:
    records: object          # torch uint8 CUDA tensor of point records
    fmt: int                 # LOD_POINTS_F32 / LOD_POINTS_F64
    n: int
    h2d_bytes: int           # file bytes streamed to the device


def _stream_to_device(f, start: int, nbytes: int, chunk: int, dst):
    """Copy file bytes [start, start + nbytes) into the CUDA tensor dst through two pinned
    staging buffers (double-buffered: the read of chunk k+1 overlaps the copy of chunk k)."""
    import torch
    stream = torch.cuda.current_stream()
    stage = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    f.seek(start)
    pos = 0
    k = 0
    while pos < nbytes:
        m = min(chunk, nbytes - pos)
        b = k & 1
        if done[b] is not None:
            done[b].synchronize()           # staging buffer b free again
        got = f.readinto(memoryview(stage[b].numpy())[:m])
        if got != m:
            raise IOError("truncated point records")
        dst[pos:pos + m].copy_(stage[b][:m], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        done[b] = ev
        pos += m
        k += 1
    torch.cuda.current_stream().synchronize()


def load_points(path, chunk_bytes: int = 64 << 20) -> DevicePoints:
    """Stream a LAS / PLY file's point records to the device and decode them there."""
    import torch
    lib = _abi.load()
    sptr = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    path = str(path)
    if path.lower().endswith(".las"):
        with open(path, "rb") as f:
            h = las_header(f)
            nbytes = h.n * h.reclen
            raw = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
            if nbytes:
                _stream_to_device(f, h.offset_to_points, nbytes, chunk_bytes, raw)
        out = torch.empty(max(h.n, 1) * 32, dtype=torch.uint8, device="cuda")
        sc, of = (C.c_double * 3)(*h.scale), (C.c_double * 3)(*h.offset)
        _abi.check(lib.lod_ingest_las(C.c_void_p(raw.data_ptr()), h.n, h.reclen, h.rgb_offset, sc, of,
                                      C.c_void_p(out.data_ptr()), sptr))
        torch.cuda.current_stream().synchronize()
        return DevicePoints(out, _abi.LOD_POINTS_F64, h.n, nbytes)
    with open(path, "rb") as f:
        head = f.read(1 << 16)
        while b"end_header" not in head:
            more = f.read(1 << 16)
            if not more:
                break
            head += more
        h = ply_header(head)
        if h.fmt == "ascii":   # text: parsed on the host, then uploaded as records
            from .device import pack_records
            f.seek(0)
            pos, col = _ply_columns(f.read(), h)
            rec, fmt = pack_records(pos, col)
            t = torch.from_numpy(rec.view(np.uint8).reshape(-1)).cuda()
            return DevicePoints(t, fmt, len(rec), t.numel())
        dt = _ply_dtype(h.props)
        nbytes = h.count * dt.itemsize
        f.seek(0, 2)
        if f.tell() - h.body_start < nbytes:
            raise IOError("truncated PLY vertex data")
        raw = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
        if nbytes:
            _stream_to_device(f, h.body_start, nbytes, chunk_bytes, raw)
    names = [p[0] for p in h.props]
    has_rgb = {"red", "green", "blue"} <= set(names)
    sel = ["x", "y", "z"] + (["red", "green", "blue"] if has_rgb else ["x", "x", "x"])
    types = (C.c_int32 * 6)(*[_PLY_CODES[dt.fields[s][0].str if dt.fields[s][0].itemsize > 1
                                         else dt.fields[s][0].str[1:]] for s in sel])
    offs = (C.c_uint32 * 6)(*[dt.fields[s][1] for s in sel])
    fmt = _abi.LOD_POINTS_F32 if all(dt.fields[a][0] == np.dtype("<f4") for a in "xyz") else _abi.LOD_POINTS_F64
    out = torch.empty(max(h.count, 1) * (16 if fmt == _abi.LOD_POINTS_F32 else 32), dtype=torch.uint8,
                      device="cuda")
    _abi.check(lib.lod_ingest_ply(C.c_void_p(raw.data_ptr()), h.count, dt.itemsize, types, offs,
                                  1 if has_rgb else 0, fmt, C.c_void_p(out.data_ptr()), sptr))
    torch.cuda.current_stream().synchronize()
    return DevicePoints(out, fmt, h.count, nbytes)


def build_file(path, config=None, strategy: str | None = None, seed: int | None = None):
    """`lodforge build` on the device (cli.py:93-118 without the file output): stream the
    file to HBM, partition, build_lod.  Returns the GpuOctree."""
    from .device import DeviceTree, make_config
    from .model import BuildConfig
    from .octree import GpuOctree
    from .sampling import build_lod
    cfg = config or BuildConfig()
    pts = load_points(path)
    if pts.n == 0:
        raise ValueError("cannot partition an empty point cloud")
    dev = DeviceTree()
    dev.split(pts.records, pts.n, pts.fmt,
              make_config(cfg.T, cfg.initial_depth, cfg.extension_depth, cfg.max_depth))
    tree = GpuOctree(dev, cfg)
    build_lod(tree, strategy, seed)
    return tree
