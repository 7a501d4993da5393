import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch, numpy as np
import bench
from paper_2302_14801_b200 import BuildConfig, Partitioner, PointCloud, build_lod
from paper_2302_14801_b200.device import DeviceTree, generate_device
import paper_2302_14801_b200.device as D
from paper_2302_14801_b200.generators import CONFIGS
kind, n, seed, _ = CONFIGS["terrain20M"]
raw = generate_device(kind, n, seed).view(torch.float32).view(n, 4)
pos32 = raw[:, :3].cpu().numpy().copy()
col = raw.view(torch.uint8).view(n, 16)[:, 12:15].cpu().numpy().copy()
pos64 = pos32.astype(np.float64)
dev = DeviceTree()
def ref():
    tree = Partitioner(PointCloud(pos64, col), BuildConfig(T=50_000), device_tree=dev).run()
    return build_lod(tree, "average", 0).node_count
for thr in (64 << 20, 4 << 20):
    D._STAGE_MIN = thr
    for _ in range(3): ref()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): ref()
    torch.cuda.synchronize()
    print("threshold", thr >> 20, "MB:", (time.perf_counter() - t0) / 5 * 1e3, "ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(5): ref()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
