"""Deterministic synthetic point clouds.

Two families:

* `reference_cloud(kind, n, seed)` restates the reference's four test presets
  (`pkg/src/lodforge/ingest.py:229-271`: uniform-cube, checker-plane, stadium,
  two-scans) bit-for-bit, so the reference's own test cases can be replayed
  against the GPU path without importing the reference.
* The BASELINE configs: `sphere`, `terrain`, `scene`, `cluster`,
  `surface`.  These emit float32 coordinates (the 16-byte device record) and
  use only IEEE-exact fp64 operations (+ - * / sqrt, floor) in a fixed order,
  so the CUDA generator in `csrc/generate.cu` reproduces them bit-for-bit for
  the billion-point configs that are generated on the device.

Every generator is counter-based (point i depends only on (seed, i)), so a
cloud can be produced in chunks, and chunk r of a sharded cloud is the same
as rows [r*n/R, (r+1)*n/R) of the whole.
"""
from __future__ import annotations

import numpy as np

from . import rng
from .model import PointCloud

REFERENCE_KINDS = ("uniform-cube", "checker-plane", "stadium", "two-scans")
SYNTHETIC_KINDS = ("sphere", "terrain", "scene", "cluster", "surface")

SCAN_A_COLOR = (200, 60, 60)   # ingest.py:15
SCAN_B_COLOR = (60, 60, 200)   # ingest.py:16
DENSE_CUBE_MIN = 0.5           # ingest.py:17
DENSE_CUBE_SIZE = 1.0 / 512.0  # ingest.py:18


# ---------------------------------------------------------------------------
# reference presets (ingest.py:229-271)
# ---------------------------------------------------------------------------


def reference_cloud(kind: str, n: int, seed: int = 0) -> PointCloud:
    """Replay `lodforge.ingest.generate(GeneratorPreset(kind, n, seed))`."""
    if kind not in REFERENCE_KINDS:
        raise ValueError(f"unknown generator kind: {kind}")
    if n < 1:
        raise ValueError("count must be >= 1")
    if kind in ("uniform-cube", "stadium"):
        raw = rng.stream(seed, 6 * n).reshape(n, 6)
        pos = rng.to_unit(raw[:, :3])
        if kind == "stadium":  # every tenth point inside a tiny dense cube (ingest.py:250-257)
            sel = np.arange(n) % 10 == 0
            pos[sel] = DENSE_CUBE_MIN + pos[sel] * DENSE_CUBE_SIZE
        col = (raw[:, 3:6] >> np.uint64(56)).astype(np.uint8)
        return PointCloud(pos, col)
    if kind == "checker-plane":  # ingest.py:238-247
        xy = rng.to_unit(rng.stream(seed, 2 * n).reshape(n, 2))
        pos = np.zeros((n, 3))
        pos[:, :2] = xy
        light = np.floor(xy * 8).astype(np.int64).sum(axis=1) % 2 == 0
        col = np.zeros((n, 3), np.uint8)
        col[light] = 255
        return PointCloud(pos, col)
    # two-scans: one jittered sheet captured twice, interleaved A,B (ingest.py:259-271)
    m = (n + 1) // 2
    raw = rng.stream(seed, 3 * m).reshape(m, 3)
    base = np.empty((m, 3))
    base[:, 0] = rng.to_unit(raw[:, 0])
    base[:, 1] = rng.to_unit(raw[:, 1])
    base[:, 2] = 0.5 + (rng.to_unit(raw[:, 2]) - 0.5) * 0.02
    pos = np.repeat(base, 2, axis=0)[:n]
    col = np.empty((2 * m, 3), np.uint8)
    col[0::2] = SCAN_A_COLOR
    col[1::2] = SCAN_B_COLOR
    return PointCloud(pos, col[:n])


# ---------------------------------------------------------------------------
# BASELINE synthetic configs (float32 coordinates)
# ---------------------------------------------------------------------------

# cluster config: 16 dense cubes of side 2^-12 plus one exact-duplicate pile.
CLUSTER_COUNT = 16
CLUSTER_SIDE = 1.0 / 4096.0
DUP_POINT = (0.25, 0.5, 0.75)

# terrain: 4 octaves of value noise on 4, 8, 16, 32-cell lattices
TERRAIN_OCTAVES = 4


def _units(seed: int, start: int, n: int, k: int) -> np.ndarray:
    """(n, k) uniforms of points start..start+n-1; point i uses stream entries [k*i, k*i+k)."""
    return rng.to_unit(rng.stream(seed, k * n, start * k)).reshape(n, k)


def _sphere_dir(u3: np.ndarray):
    """Unit direction from three uniforms: v = 2u - 1, w = v / |v| (fixed op order)."""
    vx = 2.0 * u3[:, 0] - 1.0
    vy = 2.0 * u3[:, 1] - 1.0
    vz = 2.0 * u3[:, 2] - 1.0
    r = np.sqrt((vx * vx + vy * vy) + vz * vz)
    zero = r == 0.0
    if zero.any():
        vx = np.where(zero, 1.0, vx)
        r = np.where(zero, 1.0, r)
    return vx / r, vy / r, vz / r


def _sphere_rows(u3):
    wx, wy, wz = _sphere_dir(u3)
    tx, ty, tz = 0.5 + 0.5 * wx, 0.5 + 0.5 * wy, 0.5 + 0.5 * wz
    pos = np.stack([tx, ty, tz], axis=1).astype(np.float32)
    col = np.stack([np.floor(255.0 * tx), np.floor(255.0 * ty), np.floor(255.0 * tz)], axis=1)
    return pos, col.astype(np.uint8)


def _lattice(seed: int, octave: int, ix: np.ndarray, iy: np.ndarray) -> np.ndarray:
    """Hash height in [-1, 1) at integer lattice points of one octave."""
    key = (np.uint64((seed * 8 + octave) & 0xFFFFFF) << np.uint64(40)) \
        ^ (ix.astype(np.uint64) << np.uint64(20)) ^ iy.astype(np.uint64)
    return rng.to_unit(rng.mix64_array(key)) * 2.0 - 1.0


def _terrain_rows(seed: int, u4: np.ndarray):
    x, y, jit = u4[:, 0], u4[:, 1], u4[:, 2]
    h = np.zeros_like(x)
    amp = 1.0
    for k in range(TERRAIN_OCTAVES):
        cells = float(4 << k)
        gx, gy = x * cells, y * cells
        ix, iy = np.floor(gx), np.floor(gy)
        fx, fy = gx - ix, gy - iy
        ixi, iyi = ix.astype(np.int64), iy.astype(np.int64)
        a = _lattice(seed, k, ixi, iyi)
        b = _lattice(seed, k, ixi + 1, iyi)
        c = _lattice(seed, k, ixi, iyi + 1)
        d = _lattice(seed, k, ixi + 1, iyi + 1)
        top = a + (b - a) * fx
        bot = c + (d - c) * fx
        h = h + amp * (top + (bot - top) * fy)
        amp = amp * 0.5
    z = 0.5 + 0.08 * h + 0.001 * (jit - 0.5)
    t = np.clip((z - 0.35) / 0.3, 0.0, 1.0)
    checker = (np.floor(x * 8.0) + np.floor(y * 8.0)) % 2.0 == 0.0
    col = np.stack([np.floor(255.0 * t), np.floor(255.0 * (1.0 - t)),
                    np.where(checker, 200.0, 60.0)], axis=1).astype(np.uint8)
    pos = np.stack([x, y, z], axis=1).astype(np.float32)
    return pos, col


def _cluster_corners(seed: int) -> np.ndarray:
    """Min corners of the 16 dense cubes, spread over [0.1, 0.9)^3."""
    u = rng.to_unit(rng.stream(seed ^ 0x5EED, 3 * CLUSTER_COUNT)).reshape(CLUSTER_COUNT, 3)
    return 0.1 + 0.8 * u


def scene_objects(seed: int):
    """Object table of the multi-object scene: (kind, params[7], weight) x 65.

    kind 0 = ground plane (x, y in [0, 1000), z = 0), 1 = sphere (cx, cy, cz, r),
    2 = box (cx, cy, cz, hx, hy, hz).  Weights are log-uniform in [1, 1000).
    """
    u = rng.to_unit(rng.stream(seed ^ 0x0B1EC7, 64 * 8)).reshape(64, 8)
    kinds = np.zeros(65, np.int32)
    params = np.zeros((65, 7))
    weights = np.zeros(65)
    kinds[0] = 0
    weights[0] = 2000.0
    for j in range(64):
        r = u[j]
        kinds[j + 1] = 1 if r[0] < 0.5 else 2
        cx, cy = 50.0 + 900.0 * r[1], 50.0 + 900.0 * r[2]
        ext = 5.0 + 45.0 * r[3]
        params[j + 1] = (cx, cy, ext + 300.0 * r[4], ext, ext * (0.5 + r[5]), ext * (0.5 + r[6]), 0.0)
        weights[j + 1] = np.exp(np.log(1000.0) * r[7])
    cdf = np.cumsum(weights)
    return kinds, params, cdf / cdf[-1]


def _scene_rows(seed: int, u6: np.ndarray):
    kinds, params, cdf = scene_objects(seed)
    obj = np.minimum(np.searchsorted(cdf, u6[:, 0], side="right"), len(cdf) - 1)
    k = kinds[obj]
    p = params[obj]
    pos = np.empty((len(u6), 3))
    # ground plane
    g = k == 0
    pos[g, 0] = 1000.0 * u6[g, 1]
    pos[g, 1] = 1000.0 * u6[g, 2]
    pos[g, 2] = 0.0
    # spheres
    s = k == 1
    wx, wy, wz = _sphere_dir(u6[s, 1:4])
    pos[s, 0] = p[s, 0] + p[s, 3] * wx
    pos[s, 1] = p[s, 1] + p[s, 3] * wy
    pos[s, 2] = p[s, 2] + p[s, 3] * wz
    # boxes: face = floor(6 u1), two free coords from u2, u3
    b = k == 2
    face = np.floor(6.0 * u6[b, 1]).astype(np.int64)
    a2 = 2.0 * u6[b, 2] - 1.0
    a3 = 2.0 * u6[b, 3] - 1.0
    sign = np.where(face % 2 == 0, -1.0, 1.0)
    axis = face // 2
    loc = np.empty((b.sum(), 3))
    loc[:, 0] = np.where(axis == 0, sign, a2)
    loc[:, 1] = np.where(axis == 1, sign, np.where(axis == 0, a2, a3))
    loc[:, 2] = np.where(axis == 2, sign, a3)
    pb = p[b]
    pos[b, 0] = pb[:, 0] + pb[:, 3] * loc[:, 0]
    pos[b, 1] = pb[:, 1] + pb[:, 4] * loc[:, 1]
    pos[b, 2] = pb[:, 2] + pb[:, 5] * loc[:, 2]
    base = rng.mix64_array(obj.astype(np.uint64) + np.uint64(seed * 131))
    jit = np.floor(40.0 * u6[:, 4]).astype(np.int64)
    col = np.stack([((base >> np.uint64(s_)) & np.uint64(0xBF)).astype(np.int64) + jit
                    for s_ in (8, 24, 40)], axis=1)
    return pos.astype(np.float32), col.astype(np.uint8)


def synthetic_rows(kind: str, seed: int, start: int, n: int):
    """Rows start..start+n-1 of a synthetic cloud: (float32 (n,3), uint8 (n,3))."""
    if kind == "sphere":
        return _sphere_rows(_units(seed, start, n, 3))
    if kind == "terrain":
        return _terrain_rows(seed, _units(seed, start, n, 4))
    if kind == "scene":
        return _scene_rows(seed, _units(seed, start, n, 6))
    if kind == "cluster":
        # 90% sphere surface; i % 10 == 0 -> one of 16 dense cubes of side 2^-12;
        # i % 10 == 5 and i // 10 < T + 1 -> the exact duplicate point (oversized leaf).
        u = _units(seed, start, n, 3)
        pos, col = _sphere_rows(u)
        idx = np.arange(start, start + n, dtype=np.int64)
        cl = idx % 10 == 0
        corners = _cluster_corners(seed)
        cid = (idx[cl] // 10) % CLUSTER_COUNT
        pos[cl] = (corners[cid] + CLUSTER_SIDE * u[cl]).astype(np.float32)
        dup = (idx % 10 == 5) & (idx // 10 < 50_001)
        pos[dup] = np.asarray(DUP_POINT, np.float32)
        return pos, col
    if kind == "surface":
        # sphere U terrain, interleaved: even rows sphere, odd rows terrain
        u = _units(seed, start, n, 4)
        spos, scol = _sphere_rows(u[:, :3])
        tpos, tcol = _terrain_rows(seed, u)
        odd = (np.arange(start, start + n) % 2) == 1
        spos[odd] = tpos[odd]
        scol[odd] = tcol[odd]
        return spos, scol
    raise ValueError(f"unknown synthetic kind: {kind}")


def synthetic_cloud(kind: str, n: int, seed: int, chunk: int = 1 << 22):
    """Whole synthetic cloud as (float32 (n,3) positions, uint8 (n,3) colors)."""
    pos = np.empty((n, 3), np.float32)
    col = np.empty((n, 3), np.uint8)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        pos[s:e], col[s:e] = synthetic_rows(kind, seed, s, e - s)
    return pos, col


# BASELINE.json configs -> (kind, n, seed, mode)
CONFIGS = {
    "sphere1M": ("sphere", 1_000_000, 1, "random"),
    "terrain20M": ("terrain", 20_000_000, 2, "average"),
    "scene500M": ("scene", 500_000_000, 3, "average"),
    "cluster2B": ("cluster", 2_000_000_000, 4, "average"),
    "surface4B": ("surface", 4_000_000_000, 5, "average"),
}
