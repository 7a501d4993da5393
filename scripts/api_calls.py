"""Per-call wall times of the Python API legs of bench.py's e2e_api (terrain20M), to see their
spread: fused build_lod(float32 points, colors) and partition(PointCloud(float64)) + build_lod."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2302_14801_b200 import BuildConfig, Partitioner, PointCloud, build_lod  # noqa: E402
from paper_2302_14801_b200.device import DeviceTree, generate_device  # noqa: E402
from paper_2302_14801_b200.generators import CONFIGS  # noqa: E402

kind, n, seed, _ = CONFIGS["terrain20M"]
raw = generate_device(kind, n, seed).view(torch.float32).view(n, 4)
pos32 = raw[:, :3].cpu().numpy().copy()
col = raw.view(torch.uint8).view(n, 16)[:, 12:15].cpu().numpy().copy()
pos64 = pos32.astype(np.float64)
dev = DeviceTree()
legs = {"fused_f32": lambda: build_lod(pos32, col, mode="color_filter", seed=0, device_tree=dev).node_count,
        "partition_f64": lambda: build_lod(Partitioner(PointCloud(pos64, col), BuildConfig(T=50_000),
                                                       device_tree=dev).run(), "average", 0).node_count}
for name, fn in legs.items():
    ts = []
    for _ in range(15):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(name, " ".join(f"{t:.1f}" for t in ts), "| median", round(float(np.median(ts)), 2), "ms")
