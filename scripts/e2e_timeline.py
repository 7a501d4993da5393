"""Timeline of bench.py's pipelined e2e loop (terrain20M): per-step event times of upload,
build and download on their streams, to see which engine is idle."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2302_14801_b200 import _abi  # noqa: E402
from paper_2302_14801_b200.device import DeviceTree, make_config  # noqa: E402
from paper_2302_14801_b200.generators import CONFIGS  # noqa: E402

kind, n, seed, _ = CONFIGS["terrain20M"]
d_in = bench.make_input_device(torch, kind, n, seed, start=0)
cfg = make_config(50_000)
trees = [DeviceTree(0), DeviceTree(0)]
for t in trees:
    t.build(d_in, n, _abi.LOD_POINTS_F32, cfg, 0, 0, stream=C.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
info = trees[0].info()
rec_bytes, vox_bytes = n * 16, info.n_voxels * 8
node_bytes = info.n_nodes * _abi.node_dtype().itemsize
h_in = torch.empty(rec_bytes, dtype=torch.uint8, pin_memory=True)
h_in.copy_(d_in.cpu())
d_stage = [torch.empty(rec_bytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
h_leaf = [torch.empty(rec_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
h_vox = [torch.empty(max(vox_bytes, 8), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
h_nodes = [torch.empty(max(node_bytes, 8), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
up = torch.cuda.Stream()
cs = [torch.cuda.Stream(), torch.cuda.Stream()]
lib = trees[0].lib
K = 8
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
ev = {(k, w): E() for k in range(K + 1) for w in ("u0", "u1", "b0", "b1", "d1")}
host = {}
uploaded = [torch.cuda.Event(), torch.cuda.Event()]
built = [torch.cuda.Event(), torch.cuda.Event()]
torch.cuda.synchronize()
t0 = E()
t0.record()
for b in range(2):
    built[b].record(cs[b])
with torch.cuda.stream(up):
    ev[(0, "u0")].record(up)
    d_stage[0].copy_(h_in, non_blocking=True)
    ev[(0, "u1")].record(up)
    uploaded[0].record(up)
h0 = time.perf_counter()
for k in range(K):
    b = k & 1
    host[(k, "start")] = time.perf_counter() - h0
    if k + 1 < K:
        up.wait_event(built[1 - b])
        with torch.cuda.stream(up):
            ev[(k + 1, "u0")].record(up)
            d_stage[1 - b].copy_(h_in, non_blocking=True)
            ev[(k + 1, "u1")].record(up)
            uploaded[1 - b].record(up)
    cs[b].wait_event(uploaded[b])
    sp = C.c_void_p(cs[b].cuda_stream)
    ev[(k, "b0")].record(cs[b])
    trees[b].build(d_stage[b], n, _abi.LOD_POINTS_F32, cfg, 0, 0, stream=sp)
    host[(k, "built")] = time.perf_counter() - h0
    ev[(k, "b1")].record(cs[b])
    built[b].record(cs[b])
    _abi.check(lib.lod_tree_copy_async(trees[b].h, C.c_void_p(h_leaf[b].data_ptr()), C.c_void_p(h_vox[b].data_ptr()),
                                       C.c_void_p(h_nodes[b].data_ptr()), sp))
    ev[(k, "d1")].record(cs[b])
torch.cuda.synchronize()
print(f"bytes: h2d {rec_bytes/1e6:.0f} MB, d2h {(rec_bytes+vox_bytes+node_bytes)/1e6:.0f} MB")
for k in range(K):
    r = lambda w: t0.elapsed_time(ev[(k, w)]) if (k, w) in ev else float("nan")  # noqa: E731
    print(f"step {k}: upload {r('u0'):7.2f}-{r('u1'):7.2f}  build {r('b0'):7.2f}-{r('b1'):7.2f}  download end {r('d1'):7.2f}"
          f"   host start {host[(k,'start')]*1e3:7.2f} built {host[(k,'built')]*1e3:7.2f}")
