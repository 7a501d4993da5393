"""One generated cloud, `--builds` LOD builds (for ncu launch lists / sanitizers):
    python scripts/one_build.py --config cluster2B --mode color_filter --builds 2"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cluster2B")
ap.add_argument("--mode", default="color_filter")
ap.add_argument("--points", type=int, default=0)
ap.add_argument("--builds", type=int, default=2)
a = ap.parse_args()

import torch  # noqa: E402

from paper_2302_14801_b200 import _abi  # noqa: E402
from paper_2302_14801_b200.device import DeviceTree, generate_device, make_config  # noqa: E402
from paper_2302_14801_b200.generators import CONFIGS  # noqa: E402
from paper_2302_14801_b200.sampling import _mode_code  # noqa: E402

kind, n, seed, _ = CONFIGS[a.config]
n = a.points or n
d = generate_device(kind, n, seed)
dev = DeviceTree()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(a.builds):
    dev.build(d, n, _abi.LOD_POINTS_F32, make_config(50_000), _mode_code(a.mode), 0, stream=s)
torch.cuda.synchronize()
print("ok", dev.info().n_nodes, dev.launches())
