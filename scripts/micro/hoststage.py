"""Sweep of device.host_to_device's pinned staging (buffer size, copy threads, small-array
threshold) on the array sizes the Python API uploads at terrain20M (colors 60 MB, float32
positions 240 MB, float64 positions 480 MB)."""
import time

import numpy as np
import torch

import paper_2302_14801_b200.device as D

arrs = {mb: np.random.default_rng(0).integers(0, 255, mb << 20, dtype=np.uint8) for mb in (60, 240, 480)}
for stage_mb, threads, min_mb in ((32, 8, 64), (32, 8, 4), (32, 16, 4), (64, 16, 4), (16, 16, 4), (64, 8, 4)):
    D._STAGE.clear()
    if D._POOL is not None:
        D._POOL.shutdown()
    D._POOL = None
    D._STAGE_BYTES, D._STAGE_THREADS, D._STAGE_MIN = stage_mb << 20, threads, min_mb << 20
    row = []
    for mb, a in arrs.items():
        D.host_to_device(a, 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            D.host_to_device(a, 0)
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / 5
        row.append(f"{mb} MB {sec * 1e3:6.2f} ms {a.nbytes / sec / 1e9:5.1f} GB/s")
    print(f"stage {stage_mb:3d} MB x2, {threads:2d} threads, pageable below {min_mb:3d} MB: " + " | ".join(row))
