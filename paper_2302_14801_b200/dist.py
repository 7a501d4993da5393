"""Multi-GPU LOD construction: subtree sharding, one process per GPU.

    rank r holds input rows [r*N/R, (r+1)*N/R) (contiguous shards, source-rank order =
    global input order)

    1  world cube:        local min/max            -> all-reduce MIN / MAX   (6 doubles)
    2  counting grid:     local 256^3 counts       -> all-reduce SUM         (64 MiB, NCCL)
    3  extension grids:   local counts per round   -> all-reduce SUM         (small)
    4  skeleton:          identical node table on every rank (deterministic from 2-3)
    5  plan:              cut depth d*; the inner nodes at d* are subtree units assigned
                          to ranks by LPT on point counts; leaves at depth <= d* -> rank 0
    6  exchange:          local stable distribute, leaf segments grouped by owner
                          -> all-to-all (NCCL); receivers concatenate in source-rank order,
                          which keeps every leaf's points in global input order (H3)
    7  sample:            each rank voxelizes its subtrees (depth >= d*)
    8  merge:             subtree-root voxel lists -> rank 0, which rebuilds their rank
                          structures and voxelizes depths < d*

Every step is the single-GPU algorithm restricted to a subset, so the distributed tree is
bit-identical to the single-GPU one (tests/test_dist_gpu.py checks node by node).

`RankBuilder` runs the per-rank stages through the C ABI (`lod_dist_*`); the collectives
go through a `Comm`: `NcclComm` (the library's own NCCL communicator, lod_comm_*, on the
build's stream) for real multi-GPU runs, `TorchComm` (torch.distributed, e.g. gloo: several
processes on one GPU in the tests), `LocalComm` to drive R ranks as threads of one process.
`plan_subtrees` is pure numpy (CPU-testable).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .device import DeviceTree, current_stream_ptr, make_config


# ---------------------------------------------------------------------------
# planning (host, numpy)
# ---------------------------------------------------------------------------

@dataclass
class SubtreePlan:
    cut: int                    # d*
    node_owner: np.ndarray      # int32 per node (-1: rank 0 top part)
    leaf_owner: np.ndarray      # int32 per leaf id
    roots: np.ndarray           # inner nodes at depth d* (subtree units)
    root_owner: np.ndarray      # rank per root
    load: np.ndarray            # points per rank


def subtree_points(depth, parent, leaf_node, leaf_counts):
    """Points under every node (bottom-up sums of the leaf counts)."""
    pts = np.zeros(len(depth), np.int64)
    pts[leaf_node] = leaf_counts
    by_depth = np.argsort(depth, kind="stable")
    bounds = np.searchsorted(depth[by_depth], np.arange(int(depth.max()) + 2))
    for d in range(int(depth.max()), 0, -1):
        sel = by_depth[bounds[d]:bounds[d + 1]]
        # float64 bincount is exact here (point counts < 2^53)
        pts += np.bincount(parent[sel], weights=pts[sel], minlength=len(pts)).astype(np.int64)
    return pts


def plan_subtrees(depth, parent, is_leaf, leaf_node, leaf_counts, world: int, min_units: int = 2) -> SubtreePlan:
    """Cut depth + LPT assignment of the depth-d* inner subtrees to ranks.

    depth/parent/is_leaf: per node; leaf_node: node id per leaf id; leaf_counts: global
    points per leaf id.  d* is the shallowest depth with >= min_units*world inner nodes
    (or the deepest inner depth); leaves at depth <= d* stay on rank 0, which also samples
    every inner node above d*.
    """
    depth = np.asarray(depth, np.int64)
    parent = np.asarray(parent, np.int64)
    is_leaf = np.asarray(is_leaf, bool)
    n_nodes = len(depth)
    inner = ~is_leaf
    pts = subtree_points(depth, parent, np.asarray(leaf_node), np.asarray(leaf_counts, np.int64))
    if not inner.any():
        return SubtreePlan(0, np.zeros(n_nodes, np.int32), np.zeros(len(leaf_node), np.int32),
                           np.zeros(0, np.int64), np.zeros(0, np.int32), np.array([pts[0]] + [0] * (world - 1)))
    max_inner = int(depth[inner].max())
    cut = max_inner
    for d in range(1, max_inner + 1):
        if int((inner & (depth == d)).sum()) >= min_units * world:
            cut = d
            break
    roots = np.flatnonzero(inner & (depth == cut))
    load = np.zeros(world, np.int64)
    # rank 0 also keeps the leaves above the cut and samples the top levels
    load[0] += int(pts[np.flatnonzero(is_leaf & (depth <= cut))].sum())
    root_owner = np.zeros(len(roots), np.int32)
    for i in np.argsort(-pts[roots], kind="stable"):
        r = int(np.argmin(load))
        root_owner[i] = r
        load[r] += pts[roots[i]]
    node_owner = np.full(n_nodes, -1, np.int32)
    node_owner[roots] = root_owner
    for d in range(cut + 1, int(depth.max()) + 1):
        sel = np.flatnonzero(depth == d)
        node_owner[sel] = node_owner[parent[sel]]
    node_owner[is_leaf & (depth <= cut)] = 0
    leaf_owner = node_owner[np.asarray(leaf_node)].astype(np.int32)
    return SubtreePlan(cut, node_owner, leaf_owner, roots, root_owner, load)


def exchange_layout(leaf_owner, all_counts, world, rank=None):
    """Send/receive layouts of the point exchange.

    all_counts: (R, L) points of rank r in leaf l.  For rank r: send segments (src offset in
    r's local leaf buffer, dst offset in r's send buffer, count) and send_splits[q]; recv
    segments (src offset in r's receive buffer, dst offset in r's final leaf buffer, count),
    recv_splits[q] and r's per-leaf counts.  `rank` given: that rank's layout only (what a
    rank needs: O(R L) vectorised); else the list for every rank.
    """
    all_counts = np.asarray(all_counts, np.int64)
    leaf_owner = np.asarray(leaf_owner)
    if rank is None:
        return [exchange_layout(leaf_owner, all_counts, world, r) for r in range(all_counts.shape[0])]
    R, L = all_counts.shape
    r = rank
    # send: r's leaves grouped by owner (leaf order within an owner), from r's leaf-major buffer
    order = np.argsort(leaf_owner, kind="stable")
    mine_r = all_counts[r]
    local_first = np.zeros(L, np.int64)
    local_first[1:] = np.cumsum(mine_r[:-1])
    c = mine_r[order]
    dst = np.zeros(L, np.int64)
    dst[1:] = np.cumsum(c[:-1])
    nz = c > 0
    out = {"send": (local_first[order][nz], dst[nz], c[nz]),
           "send_splits": np.bincount(leaf_owner, weights=mine_r, minlength=world).astype(np.int64)[:world]}
    # receive: the leaves r owns, every source rank's run in source-rank order (input order, H3)
    mine = np.flatnonzero(leaf_owner == r)
    A = all_counts[:, mine]                                   # (R, M)
    tot = A.sum(axis=0)
    final_first = np.zeros(len(mine), np.int64)
    final_first[1:] = np.cumsum(tot[:-1])
    recv_splits = A.sum(axis=1)
    recv_base = np.zeros(R, np.int64)
    recv_base[1:] = np.cumsum(recv_splits[:-1])
    within = np.cumsum(A, axis=1) - A                         # offset inside the source's run
    before = np.cumsum(A, axis=0) - A                         # points of lower source ranks
    nzA = A > 0
    src = (recv_base[:, None] + within)[nzA]
    dstv = (final_first[None, :] + before)[nzA]
    cnt = A[nzA]
    counts = np.zeros(L, np.uint32)
    counts[mine] = tot
    out.update({"recv": (src, dstv, cnt), "recv_splits": recv_splits, "counts": counts})
    return out


# ---------------------------------------------------------------------------
# per-rank stages (C ABI)
# ---------------------------------------------------------------------------

class _Span:
    """__cuda_array_interface__ view of a library-owned uint32 device array."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<i4", "data": (int(ptr), False),
                                         "version": 3}


def _u64(a):
    return np.ascontiguousarray(a, np.uint64)


class RankBuilder:
    def __init__(self, rank, world, device=None, dev: DeviceTree | None = None):
        self.rank, self.world = rank, world
        self.dev = dev or DeviceTree(device)
        self.lib = self.dev.lib
        self.h = self.dev.h

    def _stream(self):
        return current_stream_ptr(self.dev.device)

    def begin(self, d_records, n_local, fmt, T=50_000, initial_depth=8, extension_depth=4, max_depth=16):
        self.d_in, self.n_local, self.fmt = d_records, n_local, fmt
        self.rec_bytes = 16 if fmt == _abi.LOD_POINTS_F32 else 32
        self.cfg = make_config(T, initial_depth, extension_depth, max_depth)
        mm = (C.c_double * 6)()
        ptr = C.c_void_p(d_records.data_ptr() if n_local else 0)
        _abi.check(self.lib.lod_dist_begin(self.h, ptr, n_local, fmt, C.byref(self.cfg), mm, self._stream()))
        return np.array(mm[:3]), np.array(mm[3:])

    def count(self, n_global, world_cube):
        span = _abi.LodSpan()
        w = (C.c_double * 4)(*[float(x) for x in world_cube])
        _abi.check(self.lib.lod_dist_count(self.h, n_global, w, C.byref(span), self._stream()))
        return _Span(span.ptr, span.n)

    def extend(self):
        span = _abi.LodSpan()
        _abi.check(self.lib.lod_dist_extend(self.h, C.byref(span), self._stream()))
        return _Span(span.ptr, span.n) if span.n else None

    def skeleton(self):
        _abi.check(self.lib.lod_dist_skeleton(self.h, None, self._stream()))
        info = self.dev.info()
        self.n_leaves = info.n_leaves
        counts = np.zeros(max(info.n_leaves, 1), np.uint32)
        _abi.check(self.lib.lod_dist_leaf_counts(self.h, counts.ctypes.data_as(C.c_void_p)))
        self.nodes = self.dev.nodes()
        return counts[:info.n_leaves].copy()

    def node_arrays(self):
        nd = self.nodes
        is_leaf = (nd["flags"] & 1).astype(bool)
        leaf_node = np.flatnonzero(is_leaf)   # leaf ids are the rank of leaves in node order
        return nd["depth"].astype(np.int64), nd["parent"].astype(np.int64), is_leaf, leaf_node

    def copy_segments(self, src, dst, segs):
        s, d, c = (_u64(segs[0]), _u64(segs[1]), np.ascontiguousarray(segs[2], np.uint32))
        _abi.check(self.lib.lod_dist_copy_segments(
            self.h, C.c_void_p(src.data_ptr() if src is not None else 0),
            C.c_void_p(dst.data_ptr() if dst is not None else 0), s.ctypes.data_as(C.c_void_p),
            d.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p), len(c), self._stream()))

    def pack(self, layout):
        import torch
        send = torch.empty(max(self.n_local, 1) * self.rec_bytes, dtype=torch.uint8, device="cuda")
        self.copy_segments(None, send, layout["send"])
        return send

    def unpack_adopt(self, recv, layout):
        """Received segments straight into the tree's leaf buffer (grown first; the send buffer
        was already packed from it), adopted in place: no extra device copy."""
        n_mine = int(layout["counts"].sum())
        ptr = C.c_void_p()
        _abi.check(self.lib.lod_dist_leaf_buffer(self.h, n_mine, C.byref(ptr)))
        s, d, c = (_u64(layout["recv"][0]), _u64(layout["recv"][1]), np.ascontiguousarray(layout["recv"][2], np.uint32))
        _abi.check(self.lib.lod_dist_copy_segments(
            self.h, C.c_void_p(recv.data_ptr()), ptr, s.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p),
            c.ctypes.data_as(C.c_void_p), len(c), self._stream()))
        counts = np.ascontiguousarray(layout["counts"], np.uint32)
        _abi.check(self.lib.lod_dist_adopt(self.h, ptr, n_mine, counts.ctypes.data_as(C.c_void_p), self._stream()))

    def voxelize(self, mode, seed, mask, append=False, imports=None, imp_slot_base=0):
        mask = np.ascontiguousarray(mask, np.uint8)
        if imports:
            nodes_i = np.ascontiguousarray(imports[0], np.int32)
            counts_i = np.ascontiguousarray(imports[1], np.uint32)
            vox = imports[2]
            args = (nodes_i.ctypes.data_as(C.c_void_p), counts_i.ctypes.data_as(C.c_void_p), len(nodes_i),
                    imp_slot_base, C.c_void_p(vox.data_ptr()))
        else:
            args = (None, None, 0, 0, None)
        _abi.check(self.lib.lod_dist_voxelize(self.h, mode, int(seed) & ((1 << 64) - 1),
                                              mask.ctypes.data_as(C.c_void_p), 1 if append else 0, *args,
                                              self._stream()))

    def export_roots(self, roots):
        """Voxel runs of the given inner nodes, concatenated (device uint32 pairs) + counts:
        one library launch (lod_dist_export_roots)."""
        import torch
        roots = np.ascontiguousarray(roots, np.int32)
        counts = np.zeros(len(roots), np.uint32)
        nd = self.dev.nodes()
        total = int(nd["count"][roots].astype(np.int64).sum()) if len(roots) else 0
        out = torch.empty(max(total, 1) * 8, dtype=torch.uint8, device="cuda")
        if len(roots):
            _abi.check(self.lib.lod_dist_export_roots(self.h, roots.ctypes.data_as(C.c_void_p), len(roots),
                                                      C.c_void_p(out.data_ptr()), counts.ctypes.data_as(C.c_void_p),
                                                      self._stream()))
        return out, counts


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------

class TorchComm:
    """torch.distributed collectives (NCCL on device tensors; gloo via host copies)."""

    def __init__(self, group=None, device="cuda"):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.device = device

    def _stage(self, t):
        return t if self.nccl else t.cpu()

    def allreduce(self, t, op):
        import torch
        ops = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX}
        x = self._stage(t)
        self.dist.all_reduce(x, op=ops[op], group=self.group)
        if x is not t:
            t.copy_(x)
        return t

    def all_gather_np(self, arr):
        import torch
        x = torch.from_numpy(np.ascontiguousarray(arr)).to(self.device if self.nccl else "cpu")
        outs = [torch.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(outs, x, group=self.group)
        return np.stack([o.cpu().numpy() for o in outs])

    def all_to_all_bytes(self, send, send_splits, recv_splits):
        import torch
        total = int(sum(recv_splits))
        recv = torch.empty(max(total, 1), dtype=torch.uint8, device=self.device)
        if self.nccl:
            self.dist.all_to_all_single(recv[:total], send[:int(sum(send_splits))], [int(x) for x in recv_splits],
                                        [int(x) for x in send_splits], group=self.group)
            return recv
        # gloo: pairwise exchange through host memory
        host_send = send[:int(sum(send_splits))].cpu()
        soff = np.concatenate([[0], np.cumsum(send_splits)]).astype(np.int64)
        roff = np.concatenate([[0], np.cumsum(recv_splits)]).astype(np.int64)
        host_recv = torch.empty(max(total, 1), dtype=torch.uint8)
        reqs = []
        for q in range(self.world):
            if q == self.rank:
                host_recv[roff[q]:roff[q + 1]] = host_send[soff[q]:soff[q + 1]]
                continue
            if send_splits[q]:
                reqs.append(self.dist.isend(host_send[soff[q]:soff[q + 1]].contiguous(), q, group=self.group))
            if recv_splits[q]:
                buf = torch.empty(int(recv_splits[q]), dtype=torch.uint8)
                reqs.append((self.dist.irecv(buf, q, group=self.group), q, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                host_recv[roff[r[1]]:roff[r[1] + 1]] = r[2]
            else:
                r.wait()
        recv.copy_(host_recv)
        return recv

    def gather_bytes(self, t, nbytes):
        """Variable-size gather of device byte tensors to rank 0 (list on rank 0)."""
        import torch
        sizes = self.all_gather_np(np.array([nbytes], np.int64))[:, 0]
        mx = int(sizes.max()) or 1
        pad = torch.zeros(mx, dtype=torch.uint8, device=self.device)
        pad[:nbytes] = t[:nbytes]
        x = self._stage(pad)
        outs = [torch.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(outs, x, group=self.group)
        return [o[:int(s)].to(self.device) for o, s in zip(outs, sizes)] if self.rank == 0 else None


class NcclComm:
    """Collectives through the library's own NCCL communicator (lod_comm_*, include/lodb200.h),
    enqueued on the build's stream -- NVLink / NVSwitch, no torch.distributed on the data
    path.  torch.distributed (any backend) only broadcasts the 128-byte NCCL id at setup."""

    _DT = {"torch.int32": 0, "torch.uint32": 0, "torch.int64": 3, "torch.float64": 2}
    _OP = {"sum": 0, "min": 1, "max": 2}

    def __init__(self, rank, world, device, uid: bytes):
        self.lib = _abi.load()
        self.rank, self.world, self.nccl, self.device = rank, world, True, f"cuda:{device}"
        self.h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _abi.check(self.lib.lod_comm_init(buf, world, rank, int(device), C.byref(self.h)))

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _abi.check(_abi.load().lod_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls, device, group=None):
        import torch.distributed as dist
        obj = [cls.unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(dist.get_rank(group), dist.get_world_size(group), device, obj[0])

    def close(self):
        if self.h:
            self.lib.lod_comm_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream():
        return current_stream_ptr()

    def allreduce(self, t, op):
        _abi.check(self.lib.lod_comm_allreduce(self.h, C.c_void_p(t.data_ptr()), t.numel(), self._DT[str(t.dtype)],
                                               self._OP[op], self._stream()))
        return t

    def all_gather_np(self, arr):
        import torch
        a = np.ascontiguousarray(arr)
        x = torch.from_numpy(a.view(np.uint8).reshape(-1).copy()).to(self.device)
        out = torch.empty(x.numel() * self.world, dtype=torch.uint8, device=self.device)
        _abi.check(self.lib.lod_comm_allgather(self.h, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()),
                                               x.numel(), self._stream()))
        return out.cpu().numpy().view(a.dtype).reshape((self.world,) + a.shape)

    def all_to_all_bytes(self, send, send_splits, recv_splits):
        import torch
        sb = np.ascontiguousarray(send_splits, np.uint64)
        rb = np.ascontiguousarray(recv_splits, np.uint64)
        recv = torch.empty(max(int(rb.sum()), 1), dtype=torch.uint8, device=self.device)
        _abi.check(self.lib.lod_comm_alltoallv(self.h, C.c_void_p(send.data_ptr()), sb.ctypes.data_as(C.c_void_p),
                                               C.c_void_p(recv.data_ptr()), rb.ctypes.data_as(C.c_void_p),
                                               self._stream()))
        return recv

    def gather_bytes(self, t, nbytes):
        """Variable-size gather of device byte tensors to rank 0 (grouped send / recv to the
        root only; list of per-rank views on rank 0)."""
        import torch
        sizes = self.all_gather_np(np.array([nbytes], np.int64))[:, 0].astype(np.uint64)
        recv = None
        if self.rank == 0:
            recv = torch.empty(max(int(sizes.sum()), 1), dtype=torch.uint8, device=self.device)
        _abi.check(self.lib.lod_comm_gatherv(self.h, C.c_void_p(t.data_ptr()), int(nbytes),
                                             C.c_void_p(recv.data_ptr() if recv is not None else 0),
                                             sizes.ctypes.data_as(C.c_void_p), 0, self._stream()))
        if self.rank != 0:
            return None
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        return [recv[off[q]:off[q + 1]] for q in range(self.world)]

class LocalComm:
    """R ranks as threads of one process (tests on a single GPU): same interface as
    TorchComm, collectives through shared memory and a barrier."""

    class Group:
        def __init__(self, world):
            import threading
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, group: "LocalComm.Group", rank: int):
        self.g, self.rank, self.world, self.nccl, self.device = group, rank, group.world, True, "cuda"

    def _exchange(self, item):
        import torch
        torch.cuda.synchronize()
        self.g.slots[self.rank] = item
        self.g.barrier.wait()
        items = list(self.g.slots)
        self.g.barrier.wait()
        return items

    def allreduce(self, t, op):
        import torch
        items = self._exchange(t.clone())
        red = {"sum": lambda a, b: a + b, "min": torch.minimum, "max": torch.maximum}[op]
        acc = items[0].to(t.device)
        for x in items[1:]:
            acc = red(acc, x.to(t.device))
        t.copy_(acc)
        torch.cuda.synchronize()
        return t

    def all_gather_np(self, arr):
        return np.stack(self._exchange(np.array(arr, copy=True)))

    def all_to_all_bytes(self, send, send_splits, recv_splits):
        import torch
        items = self._exchange((send, np.asarray(send_splits, np.int64)))
        parts = []
        for r, (buf, splits) in enumerate(items):
            off = int(splits[:self.rank].sum())
            parts.append(buf[off:off + int(splits[self.rank])].to(send.device))
        out = torch.cat(parts) if parts else send[:0]
        res = torch.empty(max(out.numel(), 1), dtype=torch.uint8, device=send.device)
        res[:out.numel()] = out
        torch.cuda.synchronize()
        self._exchange(None)  # senders may reuse their buffers after this point
        return res

    def gather_bytes(self, t, nbytes):
        items = self._exchange(t[:nbytes].clone())
        return [x.to(t.device) for x in items] if self.rank == 0 else None


def simulate_distributed(records_np, fmt, world, mode, seed=0, T=50_000):
    """Run build_distributed with `world` thread-ranks on the current GPU; returns the
    RankBuilders (index = rank) and the plan.  records_np: host record array (n,) of the
    packed device format; rank r gets rows [r*n/R, (r+1)*n/R)."""
    import threading
    import torch
    n = len(records_np)
    bounds = [n * r // world for r in range(world + 1)]
    group = LocalComm.Group(world)
    dev = torch.cuda.current_device()
    out, errs = [None] * world, []

    def run(r):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(torch.cuda.Stream()):
                part = records_np[bounds[r]:bounds[r + 1]]
                d = torch.from_numpy(part.view(np.uint8).reshape(-1).copy()).cuda()
                out[r] = build_distributed(LocalComm(group, r), d, len(part), fmt, mode, seed, T)
                torch.cuda.synchronize()
        except BaseException as e:  # surface worker failures in the caller
            errs.append(e)
            group.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return [o[0] for o in out], out[0][1]


def _world_cube(lo, hi):
    """model.py:199-209 on the reduced min/max: size = max extent, 1.0 if degenerate."""
    ext = float((hi - lo).max())
    return (float(lo[0]), float(lo[1]), float(lo[2]), ext if ext > 0 else 1.0)


def build_distributed(comm: TorchComm, d_records, n_local, fmt, mode, seed=0, T=50_000, builder=None):
    """One distributed build; returns (RankBuilder, SubtreePlan).  Rank 0 ends up with the
    top levels + its subtrees, every other rank with its subtrees."""
    import torch
    rb = builder or RankBuilder(comm.rank, comm.world)
    lo, hi = rb.begin(d_records, n_local, fmt, T=T)
    lo_t = torch.tensor(lo, dtype=torch.float64, device="cuda")
    hi_t = torch.tensor(hi, dtype=torch.float64, device="cuda")
    n_t = torch.tensor([n_local], dtype=torch.int64, device="cuda")
    comm.allreduce(lo_t, "min")
    comm.allreduce(hi_t, "max")
    comm.allreduce(n_t, "sum")
    n_global = int(n_t.item())
    if n_global == 0:
        raise ValueError("cannot partition an empty point cloud")
    span = rb.count(n_global, _world_cube(lo_t.cpu().numpy(), hi_t.cpu().numpy()))
    comm.allreduce(torch.as_tensor(span, device="cuda"), "sum")
    while True:
        span = rb.extend()
        if span is None:
            break
        comm.allreduce(torch.as_tensor(span, device="cuda"), "sum")
    local_counts = rb.skeleton()
    all_counts = comm.all_gather_np(local_counts.astype(np.int64))
    depth, parent, is_leaf, leaf_node = rb.node_arrays()
    plan = plan_subtrees(depth, parent, is_leaf, leaf_node, all_counts.sum(axis=0), comm.world)
    lay = exchange_layout(plan.leaf_owner, all_counts, comm.world, comm.rank)
    send = rb.pack(lay)
    recv = comm.all_to_all_bytes(send, lay["send_splits"] * rb.rec_bytes, lay["recv_splits"] * rb.rec_bytes)
    rb.unpack_adopt(recv, lay)
    from .sampling import _mode_code
    mode_code = _mode_code(mode)
    inner = ~is_leaf
    own = inner & (plan.node_owner == comm.rank) & (depth >= plan.cut)
    rb.voxelize(mode_code, seed, own.astype(np.uint8))
    my_roots = plan.roots[plan.root_owner == comm.rank]
    vox, counts = rb.export_roots(my_roots)
    blobs = comm.gather_bytes(vox, int(counts.sum()) * 8)
    cnts = comm.gather_bytes(torch.from_numpy(counts.view(np.uint8).copy()).cuda(), counts.nbytes)
    if comm.rank == 0:
        imp_nodes, imp_counts, parts = [], [], []
        for r in range(1, comm.world):
            rr = plan.roots[plan.root_owner == r]
            cc = cnts[r].cpu().numpy().view(np.uint32)
            imp_nodes.append(rr)
            imp_counts.append(cc)
            parts.append(blobs[r][:int(cc.sum()) * 8])
        imp_nodes = np.concatenate(imp_nodes) if imp_nodes else np.zeros(0, np.int64)
        imp_counts = np.concatenate(imp_counts) if imp_counts else np.zeros(0, np.uint32)
        top = inner & (depth < plan.cut)
        vox_all = torch.cat(parts) if parts else torch.zeros(8, dtype=torch.uint8, device="cuda")
        rb.voxelize(mode_code, seed, top.astype(np.uint8), append=True,
                    imports=(imp_nodes, imp_counts, vox_all) if len(imp_nodes) else None,
                    imp_slot_base=int(len(my_roots)))
    return rb, plan
