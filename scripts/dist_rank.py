"""One rank of a multi-process distributed build (tests/test_dist_gpu.py, bench --gpus N with
--backend gloo): every rank runs build_distributed over torch.distributed (gloo: several
processes may share one GPU) and dumps its part of the tree to <out>/rank<r>.npz.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P \
        scripts/dist_rank.py --case part_uniform-cube_20000_1_T1000 --mode average --out DIR
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", required=True)
ap.add_argument("--mode", default="average")
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--out", required=True)
a = ap.parse_args()

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
from cases import by_name, make_input  # noqa: E402
from paper_2302_14801_b200.device import pack_records  # noqa: E402
from paper_2302_14801_b200.dist import TorchComm, build_distributed  # noqa: E402

case = by_name(a.case)
pos, col = make_input(case)
rec, fmt = pack_records(pos, col)
lo, hi = len(rec) * rank // world, len(rec) * (rank + 1) // world
d = torch.from_numpy(rec[lo:hi].view(np.uint8).reshape(-1).copy()).cuda()
rb, plan = build_distributed(TorchComm(), d, hi - lo, fmt, a.mode, a.seed, T=case["cfg"].get("T", 50_000))
torch.cuda.synchronize()
np.savez(os.path.join(a.out, f"rank{rank}.npz"), nodes=rb.dev.nodes(), leaf=rb.dev.leaf_records(), vox=rb.dev.voxels(),
         fmt=fmt, cut=plan.cut, node_owner=plan.node_owner)
dist.barrier()
dist.destroy_process_group()
