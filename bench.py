"""Benchmark: LOD construction points/sec (split + voxelize) on B200, BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cluster2B] [--mode color_filter]
    python bench.py --impl reference ...      # the reference's own CPU path on the host cores

One step = one full LOD build of the configured synthetic cloud: world bounds ->
counting grid -> extension rounds -> merge pyramid -> node table -> stable distribute
-> bottom-up voxelization of every inner node.  `value` is whole-job points/s with the
input resident in HBM (device time, CUDA events, max over ranks); `e2e` is the same metric
through the public C ABI from pinned HOST buffers, with the H2D copy of the input and the
D2H copy of the whole built tree (leaf points, voxels, node table) inside the timed region.

Default workload: BASELINE configs[3] = cluster2B, the largest configuration that fits one
B200 (2,000,000,000 points: 90% sphere surface, 16 dense clusters forcing extension to depth
16, an exact-duplicate oversized leaf), color filtering (reference "average"), T = 50,000,
128^3 inner grids.  For N > 1 GPUs the same fixed cloud is split N ways (rank r holds rows
[r*N_pts/N, (r+1)*N_pts/N)): strong scaling, as the north star's 2/4/8-GPU curve.  The 32-GB
input is far larger than the 126 MB L2, so no L2 flush is inserted between steps.

The CPU reference (cpu_baseline, --impl reference) is the UNMODIFIED reference (`lodforge`,
installed into baseline/_ref) when present, else the numpy oracle port, run on a subtree subset
of the same cloud: `Partitioner(subset, BuildConfig(), bounds=world)` +
`build_lod`, whose subtree is identical to the full build's (tests/test_gpu_large.py).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cluster2B")
    ap.add_argument("--mode", default="color_filter",
                    choices=["color_filter", "average", "random", "first-come", "weighted"])
    ap.add_argument("--points", type=int, default=0, help="override the config's point count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=1_500_000,
                    help="target size of the subtree subset the CPU reference builds")
    ap.add_argument("--cpu-runs", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-target", action="store_true", help="skip the north-star 1B-point scene measurement")
    ap.add_argument("--e2e-api-config", default="terrain20M",
                    help="config of the Python-API e2e leg ('' to skip)")
    ap.add_argument("--stages", action="store_true", help="also print per-stage device times to stderr")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="collectives for --gpus > 1 (gloo = host-staged, for testing on one GPU)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def make_input_device(torch, kind, n, seed, start=0):
    """Generate the synthetic cloud directly in HBM (bit-identical to generators.py)."""
    from paper_2302_14801_b200.device import generate_device
    return generate_device(kind, n, seed, start)


def measured_traffic(config, mode, n, stage):
    """DRAM bytes (read + write) per build of `stage`'s kernels, from the committed ncu launch
    list of this config (profiles/traffic.json, scripts/traffic.py); None if not profiled."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t[f"{config}:{mode}"]
        return e["stages"][stage] if e["points"] == n else None
    except Exception:
        return None


def extension_points(nodes, initial_depth=8, extension_depth=4, max_depth=16):
    """E of SURVEY 8(d): points re-read by the extension rounds = the points under every
    extension anchor (inner node at depth initial_depth + k * extension_depth < max_depth,
    partition.py:109-151), from the node table's leaf counts."""
    depth = nodes["depth"].astype(np.int64)
    cell = nodes["cell"].astype(np.int64)
    leaf = (nodes["flags"] & 1) == 1
    ldepth, lcell, lcount = depth[leaf], cell[leaf], nodes["count"][leaf].astype(np.int64)
    E = 0
    for d in range(initial_depth, max_depth, extension_depth):
        anchors = (~leaf) & (depth == d)
        if not anchors.any():
            break
        ac = cell[anchors]
        akey = (ac[:, 0] << 32) | (ac[:, 1] << 16) | ac[:, 2]
        deep = ldepth > d
        lc = lcell[deep] >> (ldepth[deep] - d)[:, None]
        lkey = (lc[:, 0] << 32) | (lc[:, 1] << 16) | lc[:, 2]
        E += int(lcount[deep][np.isin(lkey, akey)].sum())
    return E


# ---------------------------------------------------------------------------
# CPU reference (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------

def reference_impl():
    """('reference', lodforge modules) when the unmodified reference is installed in
    baseline/_ref, else ('port', the oracle)."""
    if os.path.isdir(os.path.join(REF_PATH, "lodforge")):
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        try:
            import importlib
            M, P, S = (importlib.import_module(f"lodforge.{m}") for m in ("model", "partition", "sampling"))
            from lodforge.ingest import PointCloud
            return "reference", (M, P, S, PointCloud)
        except Exception:
            pass
    from oracle import lod_oracle as O
    return "port", O


def reference_sample(config, target):
    from oracle.synth import subtree_subset
    from paper_2302_14801_b200.generators import CONFIGS
    kind, n, seed, _ = CONFIGS[config]
    return subtree_subset(kind, n, seed, target=target)


def reference_build(sample, mode, impl):
    """One timed CPU build of the subset: Partitioner(subset, cfg, bounds=world) + build_lod,
    the cli.py:105-109 scope.  Returns (seconds, outcome)."""
    kind, mod = impl
    strat = "average" if mode in ("color_filter", "average") else mode
    (lo, size) = sample["world"]
    t0 = time.perf_counter()
    outcome = "ok"
    if kind == "reference":
        M, P, S, PointCloud = mod
        cloud = PointCloud(sample["positions"], sample["colors"])
        cfg = M.BuildConfig(T=50_000, strategy=strat, seed=0)
        tree = P.Partitioner(cloud, cfg, bounds=M.AABB(tuple(lo), size)).run()
        try:
            S.build_lod(tree)
        except Exception as e:   # the 2^20 random limit (sampling.py:73-75)
            outcome = f"{type(e).__name__}: {e}"
    else:
        sp = mod.split(sample["positions"], T=50_000, bounds=(tuple(lo), size))
        try:
            mod.voxelize(sp, sample["positions"], sample["colors"], strat, 0)
        except Exception as e:
            outcome = f"{type(e).__name__}: {e}"
    return time.perf_counter() - t0, outcome


def _sample_desc(config, sample, impl_kind):
    who = ("lodforge (unmodified reference, baseline/_ref)" if impl_kind == "reference"
           else "numpy oracle port of lodforge")
    return (f"subtree subset of {config}: the {sample['count']} points of the depth-{sample['depth']} node "
            f"{tuple(sample['cell'])} in input order, Partitioner(subset, BuildConfig(T=50000), bounds=world) + "
            f"build_lod via {who}, numpy single-threaded like the reference (cli.py:246-247 ignores threads)")


def run_reference(args):
    """--impl reference: rank 0 times the reference's CPU path on a subtree subset; others exit."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    impl = reference_impl()
    sample = reference_sample(args.config, args.cpu_sample)
    for _ in range(args.warmup):
        reference_build(sample, args.mode, impl)
    times, outcome = [], "ok"
    for _ in range(args.steps):
        t, outcome = reference_build(sample, args.mode, impl)
        times.append(t)
    sec = sum(times) / len(times)
    value = sample["count"] / sec
    from paper_2302_14801_b200.generators import CONFIGS
    line = {
        "impl": "reference", "metric": f"LOD construction points/sec ({args.mode})",
        "value": value, "unit": "points/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * sec, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "points": CONFIGS[args.config][1], "mode": args.mode, "T": 50_000,
                   "grid": 128},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "host_cpu_count": os.cpu_count(),
                         "kind": impl[0], "sample": _sample_desc(args.config, sample, impl[0]),
                         "outcome": outcome},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# e2e: host buffers in, whole tree out, through the public C ABI
# ---------------------------------------------------------------------------

def _tree_bytes(dev, n):
    from paper_2302_14801_b200 import _abi
    info = dev.info()
    return n * 16 + info.n_voxels * 8 + info.n_nodes * _abi.node_dtype().itemsize


def e2e_two_trees(torch, dev, d_in, n, cfg, mode_code, steps, stream):
    """Clouds that fit twice: two trees on two streams, 2-deep pipeline (upload k+1 ||
    build k || download k-1; PCIe is full duplex)."""
    from paper_2302_14801_b200 import _abi
    from paper_2302_14801_b200.device import DeviceTree
    info = dev.info()
    rec_bytes, vox_bytes = n * 16, info.n_voxels * 8
    node_bytes = info.n_nodes * _abi.node_dtype().itemsize
    lib = dev.lib
    h_in = torch.empty(rec_bytes, dtype=torch.uint8, pin_memory=True)
    h_in.copy_(d_in)
    trees = [dev, DeviceTree(dev.device)]
    d_stage = [torch.empty(rec_bytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    h_leaf = [torch.empty(rec_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    h_vox = [torch.empty(max(vox_bytes, 8), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    h_nodes = [torch.empty(max(node_bytes, 8), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    up = torch.cuda.Stream()
    cs = [torch.cuda.Stream(), torch.cuda.Stream()]
    uploaded = [torch.cuda.Event(), torch.cuda.Event()]
    built = [torch.cuda.Event(), torch.cuda.Event()]

    def run(k_steps):
        for b in range(2):
            built[b].record(cs[b])
        with torch.cuda.stream(up):
            d_stage[0].copy_(h_in, non_blocking=True)
            uploaded[0].record(up)
        for k in range(k_steps):
            b = k & 1
            if k + 1 < k_steps:  # next input, once the build that last read the buffer is done
                up.wait_event(built[1 - b])
                with torch.cuda.stream(up):
                    d_stage[1 - b].copy_(h_in, non_blocking=True)
                    uploaded[1 - b].record(up)
            cs[b].wait_event(uploaded[b])
            sp = C.c_void_p(cs[b].cuda_stream)
            trees[b].build(d_stage[b], n, _abi.LOD_POINTS_F32, cfg, mode_code, 0, stream=sp)
            built[b].record(cs[b])
            _abi.check(lib.lod_tree_copy_async(trees[b].h, C.c_void_p(h_leaf[b].data_ptr()),
                                               C.c_void_p(h_vox[b].data_ptr()),
                                               C.c_void_p(h_nodes[b].data_ptr()), sp))
        for st in (up, cs[0], cs[1]):
            stream.wait_stream(st)

    run(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    up.wait_stream(stream)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    return (e0.elapsed_time(e1) / steps, "2 trees, 2-deep on 3 streams: upload k+1 || build k || download k-1",
            rec_bytes, _tree_bytes(dev, n))


def e2e_one_tree(torch, dev, d_in, n, cfg, mode_code, seed, steps, stream):
    """Clouds that fit once (cluster2B: ~100 GB working set): one tree, split and voxelize as
    separate ABI calls so the copies overlap the work that no longer needs their buffers --
    the next upload starts when the split has consumed the input; ONE device->host stream
    carries the leaf buffer (after the split), then the node table and the voxels (after the
    voxelize) -- the link is the bottleneck (38.9 GB down per cluster2B step), so the downloads
    queue back to back.  The next split waits only for the leaf + node downloads, and only
    before it rewrites them (lod_tree_set_output_wait); the voxel download runs under the next
    split (the split never touches the arena) and the next voxelize waits for it.  Measured
    (scripts/e2e_timeline1.py): 915 -> 860 ms per cluster2B step against the round-2 schedule,
    whose skeleton also waited for the 6.9 GB voxel download.  Both directions move as 256-MB
    pieces over two streams (two copy engines; lod_tree_copy_async splits its copies the same
    way): 45.8 -> 49.2 GB/s per direction under duplex load (scripts/micro/pcie_big.py)."""
    from paper_2302_14801_b200 import _abi
    info = dev.info()
    rec_bytes = n * 16
    lib = dev.lib
    h_in = torch.empty(rec_bytes, dtype=torch.uint8, pin_memory=True)
    h_in.copy_(d_in)
    h_leaf = torch.empty(rec_bytes, dtype=torch.uint8, pin_memory=True)
    h_vox = torch.empty(max(info.n_voxels * 8, 8), dtype=torch.uint8, pin_memory=True)
    h_nodes = torch.empty(max(info.n_nodes * _abi.node_dtype().itemsize, 88), dtype=torch.uint8, pin_memory=True)
    d_stage = d_in            # the device input buffer is the staging buffer
    up, up2, dl = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    piece = 256 << 20

    def upload():   # 256-MB pieces over two streams: two copy engines (lod_tree_copy_async does the same down)
        up2.wait_stream(up)
        for k, o in enumerate(range(0, rec_bytes, piece)):
            with torch.cuda.stream(up2 if k & 1 else up):
                d_stage[o:o + piece].copy_(h_in[o:o + piece], non_blocking=True)
        up.wait_stream(up2)
    ev_up, ev_split, ev_vox, ev_voxdl, ev_out = (torch.cuda.Event() for _ in range(5))
    sp = C.c_void_p(stream.cuda_stream)
    dlp = C.c_void_p(dl.cuda_stream)

    def run(k_steps):
        up.wait_stream(stream)
        upload()
        ev_up.record(up)
        ev_voxdl.record(dl)
        for k in range(k_steps):
            stream.wait_event(ev_up)
            if k > 0:   # the previous tree's node + leaf downloads, before the skeleton
                _abi.check(lib.lod_tree_set_output_wait(dev.h, C.c_void_p(ev_out.cuda_event)))
            dev.split(d_stage, n, _abi.LOD_POINTS_F32, cfg, stream=sp)
            ev_split.record(stream)
            if k + 1 < k_steps:             # the split consumed the input: upload the next one
                up.wait_event(ev_split)
                upload()
                ev_up.record(up)
            dl.wait_event(ev_split)         # leaf points are final after the distribute
            _abi.check(lib.lod_tree_copy_async(dev.h, C.c_void_p(h_leaf.data_ptr()), None, None, dlp))
            stream.wait_event(ev_voxdl)     # the previous voxels are downloaded: the arena is free
            dev.voxelize(mode_code, seed, stream=sp)
            ev_vox.record(stream)
            dl.wait_event(ev_vox)           # the voxelize writes the inner nodes' voxel ranges
            _abi.check(lib.lod_tree_copy_async(dev.h, None, None, C.c_void_p(h_nodes.data_ptr()), dlp))
            ev_out.record(dl)               # leaf + nodes downloaded: the next skeleton may rewrite them
            _abi.check(lib.lod_tree_copy_async(dev.h, None, C.c_void_p(h_vox.data_ptr()), None, dlp))
            ev_voxdl.record(dl)
        for st in (dl, up, up2):
            stream.wait_stream(st)

    run(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    return (e0.elapsed_time(e1) / steps,
            "1 tree: upload k+1 || voxelize k, split k+1's bounds/count/extension; one D2H stream: leaf k, "
            "nodes k, voxels k (the voxels under split k+1); copies as 256-MB pieces over two copy engines "
            "per direction",
            rec_bytes, _tree_bytes(dev, n))


def e2e_api(torch, config, mode, steps, warmup):
    """The Python drop-in from host numpy arrays: the fused
    `build_lod(points, colors, mode=...)` with float32 positions, and the reference form
    `partition(PointCloud(float64 positions, colors))` + `build_lod(tree, strategy)`.  Each
    call uploads its arrays (pinned staging) and packs them on the device; the timed region
    ends with a device->host read of the built tree's node count (the tree stays in HBM, as a
    user's lazily materialised Octree does)."""
    from paper_2302_14801_b200 import BuildConfig, Partitioner, PointCloud, build_lod
    from paper_2302_14801_b200.device import DeviceTree, generate_device
    from paper_2302_14801_b200.generators import CONFIGS
    kind, n, seed, _ = CONFIGS[config]
    raw = generate_device(kind, n, seed).view(torch.float32).view(n, 4)
    pos32 = raw[:, :3].cpu().numpy().copy()
    col = raw.view(torch.uint8).view(n, 16)[:, 12:15].cpu().numpy().copy()
    pos64 = pos32.astype(np.float64)
    del raw
    dev = DeviceTree()
    strat = "average" if mode in ("color_filter", "average") else mode
    out = {}

    def fused():
        return build_lod(pos32, col, mode=mode, seed=0, device_tree=dev).node_count

    def reference_form():
        tree = Partitioner(PointCloud(pos64, col), BuildConfig(T=50_000), device_tree=dev).run()
        return build_lod(tree, strat, 0).node_count

    for name, fn, hb in (("fused_f32", fused, 15 * n), ("partition_f64", reference_form, 27 * n)):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            fn()
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / steps
        out[name] = {"value": n / sec, "unit": "points/s", "ms_per_step": 1000 * sec, "h2d_bytes_per_step": hb,
                     "d2h_bytes_per_step": 8}
    out["config"] = config
    out["note"] = ("wall clock around the public Python API calls from host numpy arrays (upload + device pack + "
                   "build + node-count read); the built tree stays in HBM")
    return out


def north_star_target(torch, mode, n, steps):
    """BASELINE north star: >= 4 G pts/s with color filtering on 1 B200 for a 1B-point cloud
    (scene generator, first 1e9 rows; parity: tests/test_gpu_large.py test_full_cloud[scene1B])."""
    from paper_2302_14801_b200 import _abi
    from paper_2302_14801_b200.device import DeviceTree, generate_device, make_config
    from paper_2302_14801_b200.sampling import _mode_code
    d = generate_device("scene", n, 3)
    dev = DeviceTree()
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    cfg = make_config(50_000)
    for _ in range(2):
        dev.build(d, n, _abi.LOD_POINTS_F32, cfg, _mode_code(mode), 0, stream=sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        dev.build(d, n, _abi.LOD_POINTS_F32, cfg, _mode_code(mode), 0, stream=sp)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    dev.close()
    del d
    torch.cuda.empty_cache()
    return {"workload": "scene, first 1e9 rows (north-star target >= 4 G pts/s)", "points": n, "mode": mode,
            "value": n / (ms / 1000.0), "unit": "points/s", "ms_per_step": ms, "steps": steps,
            "vs_target": n / (ms / 1000.0) / 4e9}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    rank, world, local = dist_env()
    local %= max(torch.cuda.device_count(), 1)   # (>1 rank per GPU only in --backend gloo tests)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    from paper_2302_14801_b200 import _abi
    from paper_2302_14801_b200.device import DeviceTree, make_config
    from paper_2302_14801_b200.generators import CONFIGS

    kind, n_cfg, seed, _ = CONFIGS[args.config]
    n_total = args.points or n_cfg
    # strong scaling: the fixed cloud split N ways, rank r holds rows [r*N/R, (r+1)*N/R)
    start = n_total * rank // world
    n = n_total * (rank + 1) // world - start
    from paper_2302_14801_b200.sampling import _mode_code
    mode_code = _mode_code(args.mode)
    cfg = make_config(50_000)

    from paper_2302_14801_b200.device import workspace_bytes
    # lod_workspace_bytes is an upper bound (cluster2B: 153 GB estimated, 135 GB held)
    need = n * 16 + 0.75 * workspace_bytes(n, _abi.LOD_POINTS_F32, cfg, mode_code)
    free, _ = torch.cuda.mem_get_info()
    if need > free:   # e.g. surface4B (4e9 points) on one GPU: run it with --gpus >= 2
        if rank == 0:
            print(json.dumps({"metric": f"LOD construction points/sec ({args.mode})", "value": None,
                              "unit": "points/s", "n_gpus": world,
                              "config": {"workload": args.config, "points": n_total, "points_per_gpu": n},
                              "unavailable": f"{n} points per GPU need ~{need / 1e9:.0f} GB "
                                             f"(input + lod_workspace_bytes), {free / 1e9:.0f} GB free: use more GPUs"}),
                  flush=True)
        return
    d_in = make_input_device(torch, kind, n, seed, start=start)
    dev = DeviceTree(local)
    stream = torch.cuda.current_stream()
    sptr = C.c_void_p(stream.cuda_stream)
    if world > 1:
        from paper_2302_14801_b200.dist import NcclComm, RankBuilder, TorchComm, build_distributed
        # NCCL: the library's own communicator on the build stream; gloo: host-staged (tests)
        comm = None
        if args.backend == "nccl":
            try:
                comm = NcclComm.from_torch_distributed(local)
            except Exception as e:  # e.g. libnccl.so.2 not loadable by the library
                print(f"library NCCL communicator unavailable ({e}); using torch.distributed's NCCL "
                      "collectives", file=sys.stderr, flush=True)
        comm_kind = "library NCCL" if comm is not None else args.backend
        if comm is None:
            comm = TorchComm()
        rb = RankBuilder(rank, world, dev=dev)

    def step(src=None):
        src = d_in if src is None else src
        if world > 1:
            build_distributed(comm, src, n, _abi.LOD_POINTS_F32, args.mode, 0, builder=rb)
        else:
            dev.build(src, n, _abi.LOD_POINTS_F32, cfg, mode_code, 0, stream=sptr)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    info = dev.info()
    launches_per_step = dev.launches()

    # ---- timed region: K builds, inputs resident in HBM ----
    # Per-stage CUDA events (recorded by the library on the build's stream between its
    # stages) are read after every step, so the stage times -- and the roofline below --
    # are averages over exactly the timed builds.
    dev.set_timing(True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    stage_sum = [0.0] * 5
    kernel_sum = 0.0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            stage_sum = [None if a is None or b is None else a + b for a, b in zip(stage_sum, dev.stage_ms())]
            kernel_sum += dev.kernel_ms()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    stages = [None if x is None else x / args.steps for x in stage_sum]
    scatter_ms = kernel_sum / args.steps
    dev.set_timing(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    value = n_total / (ms / 1000.0)
    E = extension_points(dev.nodes())
    V = info.n_voxels
    if args.stages:
        print(f"stages ms {stages} scatter {scatter_ms} E {E} device bytes {dev.device_bytes()}", file=sys.stderr)

    # ---- e2e ----
    e2e = None
    if not args.no_e2e:
        if world == 1:
            free, _ = torch.cuda.mem_get_info()
            if free > dev.device_bytes() + 2 * n * 16 + (4 << 30):
                ems, pipeline, hb, db = e2e_two_trees(torch, dev, d_in, n, cfg, mode_code, args.steps, stream)
            else:
                ems, pipeline, hb, db = e2e_one_tree(torch, dev, d_in, n, cfg, mode_code, 0, args.steps, stream)
        else:
            h_in = torch.empty(n * 16, dtype=torch.uint8, pin_memory=True)
            h_in.copy_(d_in)
            h_leaf = torch.empty(n_total * 16 + 64, dtype=torch.uint8, pin_memory=True)
            h_vox = torch.empty(max(V * 8 * 2, 8), dtype=torch.uint8, pin_memory=True)
            h_nodes = np.zeros(info.n_nodes, _abi.node_dtype())
            lib = dev.lib

            def e2e_step():
                d_in.copy_(h_in, non_blocking=True)
                step(d_in)
                _abi.check(lib.lod_tree_copy_leaf_points(dev.h, C.c_void_p(h_leaf.data_ptr()), sptr))
                _abi.check(lib.lod_tree_copy_voxels(dev.h, C.c_void_p(h_vox.data_ptr()), sptr))
                _abi.check(lib.lod_tree_copy_nodes(dev.h, h_nodes.ctypes.data_as(C.c_void_p), sptr))

            e2e_step()
            torch.cuda.synchronize()
            torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1) / args.steps
            t = torch.tensor([ems], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
            li = dev.info()
            pipeline, hb = "serial per step", n * 16
            db = li.n_points * 16 + li.n_voxels * 8 + li.n_nodes * _abi.node_dtype().itemsize
        e2e = {"value": n_total / (ems / 1000.0), "unit": "points/s", "h2d_bytes_per_step": hb,
               "d2h_bytes_per_step": db, "ms_per_step": ems, "pipeline": pipeline}

    device_bytes = dev.device_bytes()
    api = target = None
    want_api = world == 1 and not args.no_e2e and bool(args.e2e_api_config)
    want_target = world == 1 and not args.no_target and args.config != "scene1B"
    if want_api or want_target:
        # release this build's tree, input and pinned host buffers first: the API legs allocate
        # through torch's caching allocators, and with ~170 GB of HBM (and ~70 GB of pinned host
        # memory) still held every call re-maps blocks (measured: the terrain20M API leg at
        # 1.25 / 0.61 G pts/s inside the cluster2B run against 1.63 / 1.16 G on its own)
        del d_in
        dev.close()
        torch.cuda.empty_cache()
        if hasattr(torch._C, "_host_emptyCache"):
            torch._C._host_emptyCache()
    if want_api:
        api = e2e_api(torch, args.e2e_api_config, args.mode, max(3, min(args.steps, 10)), 2)
    if want_target:
        # the north star's own target (>= 4 G pts/s color filtering on a 1B-point cloud): the
        # first 1e9 rows of the scene generator, device time of `target_steps` builds
        target = north_star_target(torch, args.mode, 1_000_000_000, 3)

    # ---- roofline (SURVEY 8(d) algorithmic bytes: B = 80 N + 16 E + 12 V) ----
    # Dominant single kernel: the distribute's K_scatter (stable counting-sort scatter), the
    # longest kernel of a build (ncu launch lists in profiles/).  Algorithmic bytes: each
    # record read once and written once, 32 B/pt, however many radix passes the
    # implementation takes (a second pass is implementation overhead, not algorithm).  Timed
    # live with CUDA events the library records around it on the build's stream.
    peak, peak_kind = hbm_peak()
    passes = max(info.radix_passes, 1)
    stage_names = ["bounds+count", "extension", "merge+nodes+targets", "distribute", "voxelize"]
    stage_bytes = [32 * n, 16 * E, 0, 32 * n, 16 * n + 12 * V]
    kern_bytes = 32 * n
    achieved = kern_bytes / (scatter_ms / 1000.0) / 1e9 if scatter_ms > 0 else 0.0
    whole_bytes = 80 * n + 16 * E + 12 * V
    mode_key = "color_filter" if args.mode in ("color_filter", "average") else args.mode
    traffic = measured_traffic(args.config, mode_key, n, "k_dist_scatter") if world == 1 else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": f"K_scatter (distribute.cu: k_dist_scatter_tma for the <= 9-bit digits of a 2-pass sort, "
                          f"k_dist_scatter_staged for one pass), {passes} radix pass(es) timed together against one "
                          f"read + one write per record",
                "algorithmic_bytes": kern_bytes, "ms_per_build": scatter_ms, "peak_source": peak_kind,
                "stages": {nm: {"ms": st, "algorithmic_bytes": b,
                                "achieved_gbs": (b / (st / 1000.0) / 1e9) if b and st else None,
                                "frac": (b / (st / 1000.0) / 1e9 / peak) if b and st else None,
                                "traffic": measured_traffic(args.config, mode_key, n, nm) if world == 1 else None}
                           for nm, st, b in zip(stage_names, stages, stage_bytes)},
                "whole_build": {"algorithmic_bytes": whole_bytes, "E": E, "V": V,
                                "achieved_gbs": whole_bytes / (ms / 1000.0) / 1e9,
                                "frac": whole_bytes / (ms / 1000.0) / 1e9 / peak}}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        impl = reference_impl()
        sample = reference_sample(args.config, args.cpu_sample)
        runs = [reference_build(sample, args.mode, impl) for _ in range(args.cpu_runs)]
        sec = statistics.median(t for t, _ in runs)
        cpu = {"value": sample["count"] / sec, "unit": "points/s", "cores": 1, "host_cpu_count": os.cpu_count(),
               "kind": impl[0], "sample": _sample_desc(args.config, sample, impl[0]) + f", median of {len(runs)}",
               "outcome": runs[-1][1], "same_config": True}

    if rank == 0:
        line = {
            "metric": f"LOD construction points/sec ({args.mode})",
            "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64-geometry/u32-counts", "data": "synthetic",
            "config": {"workload": args.config, "points": n_total, "points_per_gpu": n, "mode": args.mode,
                       "T": 50_000, "grid": 128, "l2": "input 16 B/pt x points > 126 MB L2, no flush",
                       "parallelism": f"subtree-sharded x{world} ({comm_kind} "
                                      f"all-reduce + all-to-all + rank-0 gather)"
                       if world > 1 else "single"},
            "e2e": e2e, "e2e_api": api, "gpu_launches": launches_per_step * args.steps,
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
            "stages_ms": dict(zip(stage_names, stages)),
            "tree": {"nodes": info.n_nodes, "leaves": info.n_leaves, "depth": info.depth, "voxels": V,
                     "ext_grids": info.n_ext_grids, "ext_points": E, "radix_passes": info.radix_passes,
                     "device_bytes": device_bytes},
            "north_star_target": target,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
