"""Deterministic LAS / PLY files for the ingest goldens (shared by make_ingest_golden.py, which
reads them with the REAL reference `lodforge.ingest.read_las / read_ply`, and the tests, which
decode the same bytes on the device).  Layouts follow the LAS 1.2 / 1.4 and PLY formats the
reference reads (ingest.py:55-198)."""
from __future__ import annotations

import struct

import numpy as np

LAS_RECLEN = {0: 20, 1: 28, 2: 26, 3: 34, 6: 30, 7: 36, 8: 38}     # ingest.py:55
LAS_RGB = {2: 20, 3: 28, 7: 30, 8: 30}                             # ingest.py:56
PLY_NP = {"char": "i1", "uchar": "u1", "short": "<i2", "ushort": "<u2", "int": "<i4", "uint": "<u4",
          "float": "<f4", "double": "<f8"}


def las_file(fmt: int, n: int, seed: int, pad: int = 3) -> bytes:
    """LAS 1.2 (formats 0-3, 227-byte header) or 1.4 (formats 6-8, 375-byte header with the
    64-bit point count at byte 247 and the legacy 32-bit count 0) with random integer
    coordinates over the full int32 range and random 16-bit colours."""
    rng = np.random.default_rng(seed)
    v14 = fmt >= 6
    hsize = 375 if v14 else 227
    reclen = LAS_RECLEN[fmt] + pad
    header = bytearray(hsize)
    header[0:4] = b"LASF"
    header[24], header[25] = (1, 4) if v14 else (1, 2)
    struct.pack_into("<H", header, 94, hsize)
    struct.pack_into("<I", header, 96, hsize)
    header[104] = fmt
    struct.pack_into("<H", header, 105, reclen)
    struct.pack_into("<I", header, 107, 0 if v14 else n)
    struct.pack_into("<3d", header, 131, 1e-3, 3.3e-4, 0.01)
    struct.pack_into("<3d", header, 155, 1e5, -7.5, 3.25)
    if v14:
        struct.pack_into("<Q", header, 247, n)
    rec = rng.integers(0, 256, (n, reclen), dtype=np.uint8)   # junk in the non-coordinate fields
    ints = rng.integers(-2**31, 2**31 - 1, (n, 3)).astype("<i4")
    rec[:, :12] = ints.view(np.uint8).reshape(n, 12)
    if fmt in LAS_RGB:
        b = LAS_RGB[fmt]
        rgb = rng.integers(0, 65536, (n, 3)).astype("<u2")
        rec[:, b:b + 6] = rgb.view(np.uint8).reshape(n, 6)
    return bytes(header) + rec.tobytes()


def ply_binary(ptype: str, ctype: str | None, n: int, seed: int) -> bytes:
    """binary_little_endian PLY: a leading float normal, x/y/z of `ptype`, optional colours."""
    rng = np.random.default_rng(seed)
    props = [("nx", "float")] + [(a, ptype) for a in "xyz"]
    if ctype:
        props += [(c, ctype) for c in ("red", "green", "blue")]
    rec = np.zeros(n, [(name, PLY_NP[t]) for name, t in props])
    for name, t in props:
        dt = np.dtype(PLY_NP[t])
        if name == "nx":
            rec[name] = rng.random(n)
        elif name in "xyz":
            rec[name] = (rng.random(n) * 1000 - 500) if dt.kind == "f" else rng.integers(
                np.iinfo(dt).min, np.iinfo(dt).max, n, dtype=dt)
        else:   # colours: uchar range for integer types (reference casts with astype(uint8))
            rec[name] = (rng.random(n) * 255) if dt.kind == "f" else rng.integers(
                0, min(np.iinfo(dt).max, 4000), n, dtype=dt)
    head = f"ply\nformat binary_little_endian 1.0\nelement vertex {n}\n"
    head += "".join(f"property {t} {name}\n" for name, t in props) + "element face 0\nproperty list uchar int v\n"
    head += "end_header\n"
    return head.encode() + rec.tobytes()


def ply_ascii(n: int, seed: int, rgb: bool = True) -> bytes:
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3)) * 10 - 5
    head = f"ply\nformat ascii 1.0\ncomment made by ingest_cases\nelement vertex {n}\n"
    head += "property double x\nproperty double y\nproperty double z\n"
    if rgb:
        head += "property uchar red\nproperty uchar green\nproperty uchar blue\n"
    head += "end_header\n"
    lines = []
    col = rng.integers(0, 256, (n, 3))
    for i in range(n):
        s = " ".join(repr(float(v)) for v in pos[i])
        if rgb:
            s += " " + " ".join(str(int(v)) for v in col[i])
        lines.append(s)
    return head.encode() + ("\n".join(lines) + "\n").encode()


def files():
    """name -> bytes of every ingest golden file."""
    out = {}
    for fmt in sorted(LAS_RECLEN):
        out[f"las_f{fmt}.las"] = las_file(fmt, 30_001, 100 + fmt)
    for pt, ct in [("float", "uchar"), ("double", "ushort"), ("int", "float"), ("short", "uint"),
                   ("uint", "double"), ("double", None), ("char", "char")]:
        out[f"ply_{pt}_{ct}.ply"] = ply_binary(pt, ct, 20_003, 7)
    out["ply_ascii_rgb.ply"] = ply_ascii(2_001, 8)
    out["ply_ascii_grey.ply"] = ply_ascii(999, 9, rgb=False)
    return out


# run_checks goldens (checks.py:18-92): the reference's results on reference-built trees
CHECK_CASES = [("two-scans", 120_000, 2, 2000), ("stadium", 80_000, 5, 900)]
CHECK_VARIANTS = ["split", "first-come", "average", "expected5", "tightT10"]
