"""ctypes wrapper of `oracle/synth.c` (TEST INFRASTRUCTURE: host generators for the large
BASELINE clouds, bit-identical to `paper_2302_14801_b200.generators.synthetic_rows` and to the
device generator).  Used by `tests/golden/make_subsets.py` and the CPU tests only."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "_lib", "libsynth.so")
KINDS = {"sphere": 0, "terrain": 1, "scene": 2, "cluster": 3, "surface": 4}

_lib = None


def build() -> str:
    src = os.path.join(HERE, "synth.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-f", "oracle/Makefile"], cwd=ROOT, check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(LIB)
        P = C.c_void_p
        u64, i32 = C.c_uint64, C.c_int
        lib.synth_rows.argtypes = [i32, u64, u64, u64, P, P, P]
        lib.synth_rows_idx.argtypes = [i32, u64, P, u64, P, P, P]
        lib.synth_bounds.argtypes = [i32, u64, u64, u64, P, P]
        lib.synth_bounds.restype = u64
        lib.synth_hist.argtypes = [i32, u64, u64, u64, P, P, i32, P]
        lib.synth_select.argtypes = [i32, u64, u64, u64, P, P, i32, P, P]
        _lib = lib
    return _lib


def _table(kind: str, seed: int):
    if kind != "scene":
        return None
    from paper_2302_14801_b200.generators import scene_objects
    kinds, params, cdf = scene_objects(seed)
    tab = np.zeros((65, 9))
    tab[:, 0], tab[:, 1:8], tab[:, 8] = kinds, params, cdf
    return np.ascontiguousarray(tab.reshape(-1))


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Cloud:
    """Rows of one synthetic cloud, generated on demand on all host cores."""

    def __init__(self, kind: str, seed: int):
        self.kind, self.code, self.seed = kind, KINDS[kind], seed
        self.table = _table(kind, seed)
        self.lib = load()

    def rows(self, start: int, n: int):
        pos = np.empty((n, 3), np.float32)
        col = np.empty((n, 3), np.uint8)
        self.lib.synth_rows(self.code, self.seed, start, n, _p(self.table), _p(pos), _p(col))
        return pos, col

    def rows_idx(self, idx: np.ndarray):
        idx = np.ascontiguousarray(idx, np.uint64)
        pos = np.empty((len(idx), 3), np.float32)
        col = np.empty((len(idx), 3), np.uint8)
        self.lib.synth_rows_idx(self.code, self.seed, _p(idx), len(idx), _p(self.table), _p(pos), _p(col))
        return pos, col

    def bounds(self, start: int, n: int):
        out = np.zeros(6)
        bad = self.lib.synth_bounds(self.code, self.seed, start, n, _p(self.table), _p(out))
        return out[:3], out[3:], int(bad)

    def hist(self, start: int, n: int, wb, depth: int, hist: np.ndarray):
        wb = np.ascontiguousarray(wb, np.float64)
        assert hist.dtype == np.uint64 and hist.size == 8 ** depth
        self.lib.synth_hist(self.code, self.seed, start, n, _p(self.table), _p(wb), depth, _p(hist))

    def select(self, start: int, n: int, wb, depth: int, lut: np.ndarray):
        wb = np.ascontiguousarray(wb, np.float64)
        sel = np.empty(n, np.int16)
        self.lib.synth_select(self.code, self.seed, start, n, _p(self.table), _p(wb), depth, _p(lut), _p(sel))
        return sel


def world_of(cloud: Cloud, n: int, chunk: int = 1 << 27):
    """Reference world_bounds_of (model.py:199-209) over rows [0, n): (min xyz, size)."""
    mn, mx = np.full(3, np.inf), np.full(3, -np.inf)
    for s in range(0, n, chunk):
        a, b, bad = cloud.bounds(s, min(chunk, n - s))
        if bad:
            raise ValueError("point coordinates must be finite")
        mn, mx = np.minimum(mn, a), np.maximum(mx, b)
    ext = float((mx - mn).max())
    return mn, (ext if ext > 0 else 1.0)


def subtree_subset(kind: str, n: int, seed: int, target: int = 1_500_000, T: int = 50_000,
                   chunk: int = 1 << 27):
    """A subtree subset of a synthetic cloud for the CPU reference:
    the inner node at depth 2..7 (count >= T, so inner in the full tree) whose point count is
    closest to `target`, and its points in input order.  Three passes over the rows on all host
    cores (bounds, 256^3 counts, selection).  Returns dict(positions f64, colors u8, world
    (min xyz, size), depth, cell, count)."""
    cloud = Cloud(kind, seed)
    lo, size = world_of(cloud, n, chunk)
    wb = np.array([lo[0], lo[1], lo[2], size])
    hist = np.zeros(256 ** 3, np.uint64)
    for s in range(0, n, chunk):
        cloud.hist(s, min(chunk, n - s), wb, 8, hist)
    h8 = hist.reshape(256, 256, 256)
    best = None
    for d in range(2, 8):
        k = 1 << (8 - d)
        lc = h8.reshape(1 << d, k, 1 << d, k, 1 << d, k).sum(axis=(1, 3, 5)).astype(np.int64)
        for c in np.argwhere(lc >= T):
            cnt = int(lc[tuple(c)])
            key = (abs(cnt - target), -d, tuple(int(v) for v in c))
            if best is None or key < best[0]:
                best = (key, d, tuple(int(v) for v in c), cnt)
    if best is None:   # the whole cloud is small: the root is the subset
        pos, col = cloud.rows(0, n)
        return dict(positions=pos.astype(np.float64), colors=col, world=(tuple(lo), size), depth=0,
                    cell=(0, 0, 0), count=n)
    _, d, c, cnt = best
    k = 8 - d
    lut = np.full(256 ** 3, -1, np.int16)
    lut.reshape(256, 256, 256)[c[0] << k:(c[0] + 1) << k, c[1] << k:(c[1] + 1) << k, c[2] << k:(c[2] + 1) << k] = 0
    idx = []
    for s in range(0, n, chunk):
        sel = cloud.select(s, min(chunk, n - s), wb, 8, lut)
        idx.append(np.flatnonzero(sel == 0).astype(np.uint64) + np.uint64(s))
    idx = np.concatenate(idx)
    assert len(idx) == cnt
    pos, col = cloud.rows_idx(idx)
    return dict(positions=pos.astype(np.float64), colors=col, world=(tuple(float(v) for v in lo), size), depth=d,
                cell=c, count=cnt)
