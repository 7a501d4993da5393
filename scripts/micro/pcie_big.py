"""PCIe probe at the e2e pipeline's sizes: pinned H2D / D2H of GB-sized buffers, alone and
concurrent, as one copy per direction or split into chunks over two streams per direction."""
import sys

import torch

gb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = gb << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
up = [torch.cuda.Stream() for _ in range(4)]
dn = [torch.cuda.Stream() for _ in range(4)]


def copy(dst, src, streams, chunks):
    step = (n + chunks - 1) // chunks
    for c in range(chunks):
        with torch.cuda.stream(streams[c % len(streams)]):
            dst[c * step:(c + 1) * step].copy_(src[c * step:(c + 1) * step], non_blocking=True)


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for s in up + dn:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for chunks, ns in ((1, 1), (8, 2), (32, 2), (16 * gb, 2), (16 * gb, 3), (16 * gb, 4)):
    tag = f"{chunks} chunk(s) on {ns} stream(s)"
    ms = timed(lambda: copy(d1, h1, up[:ns], chunks))
    print(f"{gb} GB h2d  {tag:24s} {ms:8.1f} ms {n / ms / 1e6:6.1f} GB/s")
    ms = timed(lambda: copy(h2, d2, dn[:ns], chunks))
    print(f"{gb} GB d2h  {tag:24s} {ms:8.1f} ms {n / ms / 1e6:6.1f} GB/s")
    ms = timed(lambda: (copy(d1, h1, up[:ns], chunks), copy(h2, d2, dn[:ns], chunks)))
    print(f"{gb} GB both {tag:24s} {ms:8.1f} ms {n / ms / 1e6:6.1f} GB/s per direction")
