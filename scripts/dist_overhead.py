"""Host overhead of the multi-GPU orchestration (dist.build_distributed) on ONE GPU: the same
cloud built through the staged path with a 1-rank NCCL communicator vs the fused lod_build,
plus a per-phase host profile of the staged build.  -> stdout (one line per measurement)."""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="scene500M")
    ap.add_argument("--points", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29611")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2302_14801_b200 import _abi
    from paper_2302_14801_b200.device import DeviceTree, generate_device, make_config
    from paper_2302_14801_b200.dist import NcclComm, RankBuilder, build_distributed
    from paper_2302_14801_b200.generators import CONFIGS
    kind, n, seed = CONFIGS[a.config][:3]
    if a.points:
        n = a.points
    buf = generate_device(kind, n, seed)
    dev = DeviceTree()
    cfg = make_config(50_000)
    for _ in range(2):
        dev.build(buf, n, _abi.LOD_POINTS_F32, cfg, _abi.LOD_MODE_AVERAGE, 0)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(a.reps):
        dev.build(buf, n, _abi.LOD_POINTS_F32, cfg, _abi.LOD_MODE_AVERAGE, 0)
    torch.cuda.synchronize()
    fused = (time.perf_counter() - t) / a.reps
    dev.close()
    comm = NcclComm.from_torch_distributed(0)
    rb = RankBuilder(0, 1)
    for _ in range(2):
        build_distributed(comm, buf, n, _abi.LOD_POINTS_F32, "color_filter", 0, builder=rb)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(a.reps):
        build_distributed(comm, buf, n, _abi.LOD_POINTS_F32, "color_filter", 0, builder=rb)
    torch.cuda.synchronize()
    staged = (time.perf_counter() - t) / a.reps
    print(f"{a.config} n={n}: fused lod_build {fused * 1e3:.1f} ms, build_distributed (1 rank, NCCL) "
          f"{staged * 1e3:.1f} ms, orchestration overhead {(staged - fused) * 1e3:.1f} ms", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    build_distributed(comm, buf, n, _abi.LOD_POINTS_F32, "color_filter", 0, builder=rb)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
