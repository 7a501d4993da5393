"""Timeline of bench.py's one-tree e2e pipeline (cluster2B by default): per-step times (ms from
the step loop start) at which each stream reaches its milestones -- upload done, split done,
leaf download done, voxelize done, voxel download done -- to see which engine is idle.

    python scripts/e2e_timeline1.py [config] [steps] [variant]

variant: base (bench.py's round-2 schedule: the next split's skeleton waits for the leaf AND
voxel+node downloads), nodesfirst (node table downloaded right after the voxelize, ahead of
the voxels; the next skeleton waits for leaf + nodes only), onestream (one D2H stream:
leaf, then nodes, then voxels; the skeleton waits for leaf + nodes).
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2302_14801_b200 import _abi  # noqa: E402
from paper_2302_14801_b200.device import DeviceTree, make_config  # noqa: E402
from paper_2302_14801_b200.generators import CONFIGS  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "cluster2B"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
variant = sys.argv[3] if len(sys.argv) > 3 else "base"
kind, n, seed, _ = CONFIGS[config]
stream = torch.cuda.current_stream()
sp = C.c_void_p(stream.cuda_stream)
d_in = bench.make_input_device(torch, kind, n, seed, start=0)
cfg = make_config(50_000)
dev = DeviceTree(0)
dev.build(d_in, n, _abi.LOD_POINTS_F32, cfg, 1, 0, stream=sp)   # sizes the tree's buffers
torch.cuda.synchronize()
info = dev.info()
lib = dev.lib
h_in = torch.empty(n * 16, dtype=torch.uint8, pin_memory=True)
h_in.copy_(d_in)
h_leaf = torch.empty(n * 16, dtype=torch.uint8, pin_memory=True)
h_vox = torch.empty(max(info.n_voxels * 8, 8), dtype=torch.uint8, pin_memory=True)
h_nodes = torch.empty(max(info.n_nodes * _abi.node_dtype().itemsize, 88), dtype=torch.uint8, pin_memory=True)
up, dl, dl2, jn = (torch.cuda.Stream() for _ in range(4))
ev_up, ev_split, ev_vox, ev_leaf, ev_voxdl, ev_out, ev_nodes = (torch.cuda.Event() for _ in range(7))
dlp, dl2p = C.c_void_p(dl.cuda_stream), C.c_void_p(dl2.cuda_stream)
T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
marks = []
e0 = T()
e0.record(stream)
up.wait_stream(stream)
with torch.cuda.stream(up):
    d_in.copy_(h_in, non_blocking=True)
    ev_up.record(up)
ev_voxdl.record(dl2)
for k in range(steps):
    m = {name: T() for name in ("up", "split", "leafdl", "vox", "voxdl")}
    stream.wait_event(ev_up)
    if k > 0:
        _abi.check(lib.lod_tree_set_output_wait(dev.h, C.c_void_p(ev_out.cuda_event)))
    dev.split(d_in, n, _abi.LOD_POINTS_F32, cfg, stream=sp)
    ev_split.record(stream)
    m["split"].record(stream)
    if k + 1 < steps:
        up.wait_event(ev_split)
        with torch.cuda.stream(up):
            d_in.copy_(h_in, non_blocking=True)
            ev_up.record(up)
            m["up"].record(up)
    dl.wait_event(ev_split)
    _abi.check(lib.lod_tree_copy_async(dev.h, C.c_void_p(h_leaf.data_ptr()), None, None, dlp))
    ev_leaf.record(dl)
    m["leafdl"].record(dl)
    stream.wait_event(ev_voxdl)
    dev.voxelize(1, 0, stream=sp)
    ev_vox.record(stream)
    m["vox"].record(stream)
    if variant == "base":
        dl2.wait_event(ev_vox)
        _abi.check(lib.lod_tree_copy_async(dev.h, None, C.c_void_p(h_vox.data_ptr()), C.c_void_p(h_nodes.data_ptr()),
                                           dl2p))
        ev_voxdl.record(dl2)
        m["voxdl"].record(dl2)
        jn.wait_event(ev_leaf)
        jn.wait_event(ev_voxdl)
    else:
        q, qp = (dl2, dl2p) if variant == "nodesfirst" else (dl, dlp)
        q.wait_event(ev_vox)
        _abi.check(lib.lod_tree_copy_async(dev.h, None, None, C.c_void_p(h_nodes.data_ptr()), qp))
        ev_nodes.record(q)
        _abi.check(lib.lod_tree_copy_async(dev.h, None, C.c_void_p(h_vox.data_ptr()), None, qp))
        ev_voxdl.record(q)
        m["voxdl"].record(q)
        jn.wait_event(ev_leaf)
        jn.wait_event(ev_nodes)
    ev_out.record(jn)
    marks.append(m)
for st in (dl, dl2, up, jn):
    stream.wait_stream(st)
e1 = T()
e1.record(stream)
torch.cuda.synchronize()
print(f"{config} [{variant}]: {steps} steps in {e0.elapsed_time(e1):.1f} ms; leaf {n * 16 / 1e9:.1f} GB, "
      f"voxels {info.n_voxels * 8 / 1e9:.2f} GB, nodes {info.n_nodes * _abi.node_dtype().itemsize / 1e6:.1f} MB")
for k, m in enumerate(marks):
    row = []
    for name in ("split", "up", "leafdl", "vox", "voxdl"):
        try:
            row.append(f"{name} {e0.elapsed_time(m[name]):8.1f}")
        except (RuntimeError, ValueError):
            row.append(f"{name} {'-':>8}")
    print(f"step {k}: " + "  ".join(row))
