"""Cost of page-locking a caller's numpy array in place (cudaHostRegister) + a direct DMA, against
the pinned-staging upload device.host_to_device uses (host memcpy into two 32-MB pinned buffers
by 8 threads, overlapped with the DMA)."""
import time

import numpy as np
import torch

from paper_2302_14801_b200.device import host_to_device

cudart = torch.cuda.cudart()
for mb in (64, 540, 2048):
    a = np.random.default_rng(0).integers(0, 255, mb << 20, dtype=np.uint8)
    d = torch.empty(a.nbytes, dtype=torch.uint8, device="cuda")
    host_to_device(a, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        host_to_device(a, 0)
    torch.cuda.synchronize()
    staged = (time.perf_counter() - t0) / 3
    regs, unregs, dmas = [], [], []
    for _ in range(3):
        t0 = time.perf_counter()
        r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        t1 = time.perf_counter()
        d.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        cudart.cudaHostUnregister(a.ctypes.data)
        t3 = time.perf_counter()
        regs.append(t1 - t0), dmas.append(t2 - t1), unregs.append(t3 - t2)
    print(f"{mb:5d} MB  staged {staged * 1e3:7.2f} ms ({a.nbytes / staged / 1e9:5.1f} GB/s) | register {min(regs) * 1e3:6.2f} ms"
          f"  dma {min(dmas) * 1e3:6.2f} ms  unregister {min(unregs) * 1e3:6.2f} ms  (rc {int(r)})  -> "
          f"{a.nbytes / (min(regs) + min(dmas) + min(unregs)) / 1e9:5.1f} GB/s")
