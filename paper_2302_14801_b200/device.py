"""Device-side tree handle: uploads point records, runs the C ABI, copies results back.

torch is used only for device buffers and the current CUDA stream; every byte of
LOD work runs in `liblodb200.so`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import LOD_POINTS_F32, LOD_POINTS_F64, LodConfig, LodTreeInfo

REC_F32 = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("rgba", "u1", 4)])
REC_F64 = np.dtype([("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("rgba", "u1", 4), ("pad", "u1", 4)])


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2302_14801_b200 needs a CUDA device (no CPU fallback)")
    return torch


def f32_exact(positions: np.ndarray) -> bool:
    """True when float64 coordinates survive a float32 round trip (then 16-byte records are exact)."""
    p = np.asarray(positions, np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        return bool(np.array_equal(p.astype(np.float32).astype(np.float64), p))


def pack_records(positions, colors, fmt: int | None = None):
    """Host record array for `positions` (n,3) and `colors` (n,3) u8; picks F32 when exact."""
    pos = np.asarray(positions)
    col = np.asarray(colors, np.uint8).reshape(-1, 3)
    if fmt is None:
        fmt = LOD_POINTS_F32 if (pos.dtype == np.float32 or f32_exact(pos)) else LOD_POINTS_F64
    rec = np.zeros(len(col), REC_F32 if fmt == LOD_POINTS_F32 else REC_F64)
    rec["x"], rec["y"], rec["z"] = pos[:, 0], pos[:, 1], pos[:, 2]
    rec["rgba"][:, :3] = col
    return rec, fmt


def unpack_records(raw: np.ndarray, fmt: int):
    rec = raw.view(REC_F32 if fmt == LOD_POINTS_F32 else REC_F64)
    pos = np.stack([rec["x"], rec["y"], rec["z"]], axis=1).astype(np.float64)
    col = np.ascontiguousarray(rec["rgba"][:, :3])
    return pos, col


_STAGE = {}          # device -> (pinned staging buffers, events, copy stream, lock)
_STAGE_BYTES = 32 << 20
_STAGE_THREADS = 8
_STAGE_MIN = 4 << 20    # smaller arrays: one pageable copy (pageable runs at ~11 GB/s: 60 MB 6.0 -> 2.3 ms staged)
_POOL = None
_STAGE_LOCK = None


def host_to_device(arr: np.ndarray, device: int):
    """Contiguous host array -> uint8 device tensor of its bytes.  Large arrays are copied
    through two pinned 32-MB staging buffers: the host copy into one (split over 8 threads;
    numpy copies release the GIL) overlaps the DMA of the other.  Sizes, threads and the
    threshold come from a sweep on the B200 box (scripts/micro/hoststage.py; 16 threads or
    64-MB buffers were slower, page-locking the caller's array in place costs more than the
    copy: scripts/micro/hostreg.py)."""
    global _POOL
    torch = _torch()
    src = np.ascontiguousarray(arr).reshape(-1).view(np.uint8)
    nb = src.nbytes
    out = torch.empty(max(nb, 1), dtype=torch.uint8, device=f"cuda:{device}")
    if nb <= _STAGE_MIN:
        if nb:
            out.copy_(torch.from_numpy(src))
        return out[:nb]
    global _STAGE_LOCK
    import threading
    if _STAGE_LOCK is None:
        _STAGE_LOCK = threading.Lock()
    with _STAGE_LOCK:   # one staging ring per device, shared by every caller thread
        if device not in _STAGE:
            bufs = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            _STAGE[device] = (bufs, [torch.cuda.Event(), torch.cuda.Event()], torch.cuda.Stream(device),
                              threading.Lock())
        if _POOL is None:
            import concurrent.futures as cf
            _POOL = cf.ThreadPoolExecutor(_STAGE_THREADS)
    bufs, evs, cs, lock = _STAGE[device]
    with lock:
        cs.wait_stream(torch.cuda.current_stream(device))
        for k, off in enumerate(range(0, nb, _STAGE_BYTES)):
            m = min(_STAGE_BYTES, nb - off)
            b = k & 1
            evs[b].synchronize()                      # the DMA that last read this buffer is done
            dst = bufs[b].numpy()
            q = (m + _STAGE_THREADS - 1) // _STAGE_THREADS
            parts = [(a, min(m, a + q)) for a in range(0, m, q)]
            list(_POOL.map(lambda ab: np.copyto(dst[ab[0]:ab[1]], src[off + ab[0]:off + ab[1]]), parts))
            with torch.cuda.stream(cs):
                out[off:off + m].copy_(bufs[b][:m], non_blocking=True)
                evs[b].record(cs)
        torch.cuda.current_stream(device).wait_stream(cs)
    return out[:nb]


def generate_device(kind: str, n: int, seed: int, start: int = 0, out=None):
    """Rows [start, start+n) of a BASELINE synthetic cloud generated in HBM as 16-B F32 records
    (uint8 torch tensor of n*16 bytes; `lod_generate`, bit-identical to generators.py)."""
    torch = _torch()
    from .generators import scene_objects
    lib = _abi.load()
    buf = torch.empty(n * 16, dtype=torch.uint8, device="cuda") if out is None else out
    table = None
    if kind == "scene":
        kinds, params, cdf = scene_objects(seed)
        tab = np.zeros((65, 9))
        tab[:, 0], tab[:, 1:8], tab[:, 8] = kinds, params, cdf
        table = torch.from_numpy(tab.reshape(-1)).to(buf.device)
    stream = C.c_void_p(torch.cuda.current_stream(buf.device).cuda_stream)
    tptr = C.cast(C.c_void_p(table.data_ptr()), C.POINTER(C.c_double)) if table is not None else None
    chunk = 1 << 28
    with torch.cuda.device(buf.device):   # lod_generate launches on the current device
        for s in range(0, n, chunk):
            m = min(chunk, n - s)
            _abi.check(lib.lod_generate(kind.encode(), seed, start + s, m, C.c_void_p(buf.data_ptr() + s * 16), tptr,
                                        stream))
    torch.cuda.current_stream(buf.device).synchronize()
    return buf


def make_config(T=50_000, initial_depth=8, extension_depth=4, max_depth=16) -> LodConfig:
    return LodConfig(int(T), int(initial_depth), int(extension_depth), int(max_depth))


def current_stream_ptr(device: int | None = None):
    """torch's current stream ON `device` (default: the current device) as a void*."""
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_uint64, C.c_int, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p)
_ALLOCATOR = None


def use_torch_allocator(enable: bool = True):
    """Route the library's device allocations through torch's caching allocator
    (lod_set_allocator), so torch.cuda.memory_allocated() and the framework's OOM handling see
    the HBM the trees hold.  On by default for trees made through this package; set
    LODB200_CUDA_MALLOC=1 to keep plain cudaMalloc."""
    global _ALLOCATOR
    torch = _torch()
    lib = _abi.load()
    if not enable:
        _abi.check(lib.lod_set_allocator(None, None, None))
        _ALLOCATOR = None
        return

    def alloc(nbytes, device, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), int(device))
        except Exception:   # out of memory: the library reports a CUDA allocation error
            return None

    def free(ptr, nbytes, device, ctx):
        try:
            torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:   # interpreter shutdown: torch may already be gone
            pass

    _ALLOCATOR = (_ALLOC_FN(alloc), _FREE_FN(free))   # keep the thunks alive
    _abi.check(lib.lod_set_allocator(C.cast(_ALLOCATOR[0], C.c_void_p), C.cast(_ALLOCATOR[1], C.c_void_p), None))


def workspace_bytes(n: int, fmt: int = LOD_POINTS_F32, config: LodConfig | None = None, mode: int = 1) -> int:
    """lod_workspace_bytes: planning estimate of one build's device bytes."""
    out = C.c_uint64()
    cfg = config or make_config()
    _abi.check(_abi.load().lod_workspace_bytes(int(n), int(fmt), C.byref(cfg), int(mode), C.byref(out)))
    return int(out.value)


class DeviceTree:
    """One `lod_tree` handle (grow-only device buffers reused across builds)."""

    def __init__(self, device: int | None = None):
        import os
        torch = _torch()
        self.lib = _abi.load()
        if _ALLOCATOR is None and os.environ.get("LODB200_CUDA_MALLOC", "0") != "1":
            use_torch_allocator(True)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.h = self.lib.lod_tree_create(self.device)
        if not self.h:
            raise RuntimeError(self.lib.lod_last_error().decode())
        self._input = None
        self.generation = 0   # bumped by every split: trees built earlier on this handle are stale

    def close(self):
        """Free the tree's device buffers now (also done when the handle is collected)."""
        h = getattr(self, "h", None)
        if h:
            try:
                self.lib.lod_tree_destroy(h)
            except Exception:
                pass
            self.h = None

    def __del__(self):
        self.close()

    # -- uploads -------------------------------------------------------------
    def upload(self, positions, colors, fmt: int | None = None):
        """Host (n,3) float32/float64 positions + (n,3) uint8 colours -> device records.

        The arrays go to HBM as they are (host_to_device: pinned staging, parallel host copies)
        and are packed there (`lod_pack_points`): F32 records when the coordinates are float32
        or float64 values exact in float32, else F64 records.  No per-point host work."""
        torch = _torch()
        pos = np.asarray(positions)
        if pos.dtype != np.float32 and pos.dtype != np.float64:
            pos = pos.astype(np.float64)
        pos = np.ascontiguousarray(pos).reshape(-1, 3)
        col = np.ascontiguousarray(np.asarray(colors, np.uint8)).reshape(-1, 3)
        n = len(pos)
        if len(col) != n:
            raise ValueError("positions/colors length mismatch")
        dev = f"cuda:{self.device}"
        f64 = pos.dtype == np.float64
        d_xyz = host_to_device(pos, self.device)
        d_rgb = host_to_device(col, self.device)
        out = torch.empty(max(n, 1) * (32 if (f64 and fmt != LOD_POINTS_F32) else 16), dtype=torch.uint8, device=dev)
        chosen = C.c_int(-1)
        with torch.cuda.device(self.device):   # lod_pack_points runs on the current device
            _abi.check(self.lib.lod_pack_points(C.c_void_p(d_xyz.data_ptr()), 1 if f64 else 0,
                                                C.c_void_p(d_rgb.data_ptr()), n, -1 if fmt is None else int(fmt),
                                                C.c_void_p(out.data_ptr()), C.byref(chosen),
                                                current_stream_ptr(self.device)))
        fmt = chosen.value
        return out[: n * (16 if fmt == LOD_POINTS_F32 else 32)], fmt, n

    # -- C ABI calls -----------------------------------------------------------
    def split(self, d_records, n: int, fmt: int, config: LodConfig, bounds=None, stream=None):
        b = None
        if bounds is not None:
            b = (C.c_double * 4)(*[float(x) for x in bounds])
        self.generation += 1
        self._input = d_records  # keep alive for the duration of the call
        _abi.check(self.lib.lod_split(self.h, C.c_void_p(d_records.data_ptr()), n, fmt, b, C.byref(config),
                                      stream if stream is not None else current_stream_ptr(self.device)))
        self._input = None

    def voxelize(self, mode: int, seed: int, stream=None):
        _abi.check(self.lib.lod_voxelize(self.h, mode, int(seed) & ((1 << 64) - 1),
                                         stream if stream is not None else current_stream_ptr(self.device)))

    def build(self, d_records, n: int, fmt: int, config: LodConfig, mode: int, seed: int, stream=None):
        self.generation += 1
        _abi.check(self.lib.lod_build(self.h, C.c_void_p(d_records.data_ptr()), n, fmt, C.byref(config), mode,
                                      int(seed) & ((1 << 64) - 1),
                                      stream if stream is not None else current_stream_ptr(self.device)))

    def info(self) -> LodTreeInfo:
        out = LodTreeInfo()
        _abi.check(self.lib.lod_tree_get_info(self.h, C.byref(out)))
        return out

    def nodes(self) -> np.ndarray:
        info = self.info()
        arr = np.zeros(info.n_nodes, _abi.node_dtype())
        _abi.check(self.lib.lod_tree_copy_nodes(self.h, arr.ctypes.data_as(C.c_void_p), current_stream_ptr(self.device)))
        return arr

    def leaf_records(self) -> np.ndarray:
        info = self.info()
        size = 16 if info.point_format == LOD_POINTS_F32 else 32
        raw = np.empty(info.n_points * size, np.uint8)
        _abi.check(self.lib.lod_tree_copy_leaf_points(self.h, raw.ctypes.data_as(C.c_void_p), current_stream_ptr(self.device)))
        return raw

    def voxels(self) -> np.ndarray:
        info = self.info()
        raw = np.empty((info.n_voxels, 2), np.uint32)
        if info.n_voxels:
            _abi.check(self.lib.lod_tree_copy_voxels(self.h, raw.ctypes.data_as(C.c_void_p), current_stream_ptr(self.device)))
        return raw

    # -- stage exports (the reference Partitioner's intermediate arrays) ------------------

    def point_keys(self, n: int) -> np.ndarray:
        """Finest main-grid key (cx * dim + cy) * dim + cz of each input point (count stage)."""
        out = np.empty(n, np.uint32)
        _abi.check(self.lib.lod_tree_copy_point_keys(self.h, out.ctypes.data_as(C.c_void_p),
                                                     current_stream_ptr(self.device)))
        return out

    def pyramids(self) -> np.ndarray:
        """Every counting pyramid of the build, u32 per cell (main at 0, extensions after)."""
        n = C.c_uint64()
        _abi.check(self.lib.lod_tree_copy_pyramids(self.h, None, C.byref(n), None))
        out = np.empty(n.value, np.uint32)
        _abi.check(self.lib.lod_tree_copy_pyramids(self.h, out.ctypes.data_as(C.c_void_p), C.byref(n),
                                                   current_stream_ptr(self.device)))
        return out

    def ext_grids(self):
        """The extension grids in creation order: list of LodExtGrid."""
        n = C.c_uint32()
        _abi.check(self.lib.lod_tree_ext_grids(self.h, None, C.byref(n), None))
        arr = (_abi.LodExtGrid * max(n.value, 1))()
        if n.value:
            _abi.check(self.lib.lod_tree_ext_grids(self.h, C.cast(arr, C.c_void_p), C.byref(n),
                                                   current_stream_ptr(self.device)))
        return list(arr[:n.value])

    def ext_points(self):
        """(input index, depth-16 cell (n, 3)) of every point inside an extension grid."""
        n = C.c_uint64()
        _abi.check(self.lib.lod_tree_ext_points(self.h, None, None, C.byref(n), None))
        idx = np.empty(n.value, np.uint32)
        packed = np.empty(n.value, np.uint64)
        if n.value:
            _abi.check(self.lib.lod_tree_ext_points(self.h, idx.ctypes.data_as(C.c_void_p),
                                                    packed.ctypes.data_as(C.c_void_p), C.byref(n),
                                                    current_stream_ptr(self.device)))
        cells = np.stack([packed & 0xFFFF, (packed >> 16) & 0xFFFF, packed >> 32], axis=1).astype(np.int64)
        return idx.astype(np.int64), cells

    def leaf_range(self, first: int, count: int) -> np.ndarray:
        """Raw records [first, first+count) of the leaf buffer (one node's points)."""
        size = 16 if self.info().point_format == LOD_POINTS_F32 else 32
        raw = np.empty(count * size, np.uint8)
        _abi.check(self.lib.lod_tree_copy_range(self.h, 0, first, count, raw.ctypes.data_as(C.c_void_p),
                                                current_stream_ptr(self.device)))
        return raw

    def voxel_range(self, first: int, count: int) -> np.ndarray:
        """(count, 2) u32 {key, rgb} voxels [first, first+count) in stored order."""
        raw = np.empty((count, 2), np.uint32)
        _abi.check(self.lib.lod_tree_copy_range(self.h, 1, first, count, raw.ctypes.data_as(C.c_void_p),
                                                current_stream_ptr(self.device)))
        return raw

    def device_ptrs(self):
        lp, vp = C.c_void_p(), C.c_void_p()
        _abi.check(self.lib.lod_tree_leaf_points(self.h, C.byref(lp)))
        if self.info().voxel_mode >= 0:
            _abi.check(self.lib.lod_tree_voxels(self.h, C.byref(vp)))
        return lp.value, vp.value

    def set_timing(self, on: bool):
        _abi.check(self.lib.lod_set_timing(self.h, 1 if on else 0))

    def stage_ms(self):
        out = (C.c_float * 5)()
        _abi.check(self.lib.lod_tree_stage_ms(self.h, out))
        return [None if x != x else float(x) for x in out]   # NaN: stage not bracketed

    def kernel_ms(self) -> float:
        """Device ms of the distribute's K_scatter (all passes) in the last timed build."""
        out = (C.c_float * 1)()
        _abi.check(self.lib.lod_tree_kernel_ms(self.h, out))
        return float(out[0])

    def launches(self) -> int:
        return int(self.lib.lod_tree_launches(self.h))

    def device_bytes(self) -> int:
        return int(self.lib.lod_tree_device_bytes(self.h))
