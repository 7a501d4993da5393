"""Benchmark: LOD construction points/sec (split + voxelize) on B200, BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config terrain20M] [--mode color_filter]
    python bench.py --impl reference ...      # the reference's CPU path (oracle port) on host cores

One step = one full LOD build of the configured synthetic cloud: world bounds ->
counting grid -> extension rounds -> merge pyramid -> node table -> stable distribute
-> bottom-up voxelization of every inner node.  `value` is whole-job points/s with the
input resident in HBM (device time, CUDA events, max over ranks); `e2e` is the same metric
through the public API from pinned HOST buffers, with the H2D copy of the input and the
D2H copy of the whole built tree (leaf points, voxels, node table) inside the timed region.

Default workload (N=1): BASELINE configs[1] = 20M-point terrain heightfield, color
filtering (reference "average"), T = 50,000, 128^3 inner grids.  The 320 MB input is
larger than the 126 MB L2, so no L2 flush is inserted between steps.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="terrain20M")
    ap.add_argument("--mode", default="color_filter",
                    choices=["color_filter", "average", "random", "first-come", "weighted"])
    ap.add_argument("--points", type=int, default=0, help="override the config's point count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=2_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
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
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


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
    from paper_2302_14801_b200 import _abi
    from paper_2302_14801_b200.generators import scene_objects
    lib = _abi.load()
    buf = torch.empty(n * 16, dtype=torch.uint8, device="cuda")
    table = None
    if kind == "scene":
        kinds, params, cdf = scene_objects(seed)
        tab = np.zeros((65, 9))
        tab[:, 0], tab[:, 1:8], tab[:, 8] = kinds, params, cdf
        table = torch.from_numpy(tab.reshape(-1)).cuda()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    tptr = C.cast(C.c_void_p(table.data_ptr()), C.POINTER(C.c_double)) if table is not None else None
    chunk = 1 << 28
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        _abi.check(lib.lod_generate(kind.encode(), seed, start + s, m, C.c_void_p(buf.data_ptr() + s * 16), tptr,
                                    stream))
    torch.cuda.synchronize()
    return buf


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


def cpu_reference_rate(kind, seed, sample, mode, steps=1):
    """The reference algorithm on the host (oracle port, numpy, 1 core): points/s on a sample."""
    from oracle import lod_oracle as O
    from paper_2302_14801_b200.generators import synthetic_rows
    pos, col = synthetic_rows(kind, seed, 0, sample)
    pos64 = pos.astype(np.float64)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        sp = O.split(pos64)
        O.voxelize(sp, pos64, col, mode, 0)
        times.append(time.perf_counter() - t0)
    return sample / statistics.median(times), times


def run_reference(args):
    """--impl reference: rank 0 times the reference's CPU path (oracle port); others exit."""
    rank, world, _ = dist_env()
    from paper_2302_14801_b200.generators import CONFIGS
    kind, n, seed, _ = CONFIGS[args.config]
    if rank != 0:
        return
    sample = min(args.cpu_sample, n)
    mode = "average" if args.mode in ("color_filter", "average") else args.mode
    for _ in range(args.warmup):
        cpu_reference_rate(kind, seed, min(sample, 100_000), mode)
    rates, times = [], []
    for _ in range(args.steps):
        r, t = cpu_reference_rate(kind, seed, sample, mode)
        rates.append(r)
        times += t
    value = sample / (sum(times) / len(times))
    line = {
        "impl": "reference", "metric": f"LOD construction points/sec ({args.mode})",
        "value": value, "unit": "points/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "points": n, "mode": args.mode, "T": 50_000, "grid": 128},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "kind": "port",
                         "sample": f"first {sample} points of {args.config} per step (numpy oracle port of "
                                   f"lodforge partition + build_lod, single-threaded like the reference)"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    n = args.points or n_cfg
    from paper_2302_14801_b200.sampling import _mode_code
    mode_code = _mode_code(args.mode)
    cfg = make_config(50_000)

    # weak scaling: rank r holds rows [r*n, (r+1)*n) of one N*n-point cloud; for N > 1 the
    # ranks build ONE tree together (dist.py: all-reduced grids, subtree all-to-all, rank-0 merge)
    d_in = make_input_device(torch, kind, n, seed, start=rank * n)
    dev = DeviceTree(local)
    stream = torch.cuda.current_stream()
    sptr = C.c_void_p(stream.cuda_stream)
    if world > 1:
        from paper_2302_14801_b200.dist import RankBuilder, TorchComm, build_distributed
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
            stage_sum = [a + b for a, b in zip(stage_sum, dev.stage_ms())]
            kernel_sum += dev.kernel_ms()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    stages = [x / args.steps for x in stage_sum]
    scatter_ms = kernel_sum / args.steps
    dev.set_timing(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    value = n * world / (ms / 1000.0)

    # ---- e2e: host buffers in, whole tree out, through the public C ABI ----
    # Every step uploads its input from pinned host memory and downloads the whole built
    # tree (leaf points, voxels, node table).  On one GPU the steps are pipelined two deep
    # on separate streams -- upload of step k+1 || build of step k || download of step k-1
    # (PCIe is full duplex; the library's lod_tree_copy_async enqueues the downloads) -- the
    # way a stream of clouds would be processed.  N > 1 ranks run the steps serially.
    e2e = None
    if not args.no_e2e:
        rec_bytes = n * 16
        vox_bytes = info.n_voxels * 8
        node_bytes = info.n_nodes * _abi.node_dtype().itemsize
        h_in = torch.empty(rec_bytes, dtype=torch.uint8, pin_memory=True)
        h_in.copy_(d_in.cpu())
        lib = dev.lib
        if world == 1:
            trees = [dev, DeviceTree(local)]
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
            run(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1) / args.steps
            pipeline = "2-deep on 3 streams: upload k+1 || build k || download k-1"
        else:
            h_leaf = torch.empty(rec_bytes * 2, dtype=torch.uint8, pin_memory=True)
            h_vox = torch.empty(max(vox_bytes, 8) * 2, dtype=torch.uint8, pin_memory=True)
            h_nodes = np.zeros(info.n_nodes, _abi.node_dtype())
            d_stage = torch.empty(rec_bytes, dtype=torch.uint8, device="cuda")

            def e2e_step():
                d_stage.copy_(h_in, non_blocking=True)
                step(d_stage)
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
            pipeline = "serial per step"
        e2e = {"value": n * world / (ems / 1000.0), "unit": "points/s", "h2d_bytes_per_step": rec_bytes,
               "d2h_bytes_per_step": rec_bytes + vox_bytes + node_bytes, "ms_per_step": ems,
               "pipeline": pipeline}

    # ---- roofline ----
    # Dominant single kernel: the distribute's K_scatter (stable counting-sort scatter), the
    # longest kernel of a build (ncu launch lists in profiles/).  Its algorithmic bytes per
    # pass: every record read once and written once (32 B/pt).  Timed live with CUDA events
    # the library records around it on the build's stream, averaged over the timed builds.
    # Per stage: bounds 16N + count 16N, extension 16E, distribute 32N,
    # voxelize 16N + 12V (each voxel written and read once as a 6-B record); the skeleton
    # (merge / nodes / targets) is N-independent.
    peak, peak_kind = hbm_peak()
    V = info.n_voxels
    passes = max(info.radix_passes, 1)
    stage_names = ["bounds+count", "extension", "merge+nodes+targets", "distribute", "voxelize"]
    stage_bytes = [32 * n, 16 * n if info.n_ext_grids else 0, 0, 32 * n, 16 * n + 12 * V]
    kern_bytes = 32 * n * passes
    achieved = kern_bytes / (scatter_ms / 1000.0) / 1e9 if scatter_ms > 0 else 0.0
    whole_bytes = 80 * n + 12 * V
    traffic = measured_traffic(args.config, args.mode, n, "k_dist_scatter") if world == 1 else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": f"K_scatter (distribute.cu: k_dist_scatter_staged for f32 records), {passes} pass(es)",
                "algorithmic_bytes": kern_bytes, "ms_per_build": scatter_ms, "peak_source": peak_kind,
                "stages": {nm: {"ms": st, "algorithmic_bytes": b,
                                "achieved_gbs": (b / (st / 1000.0) / 1e9) if b and st > 0 else None,
                                "traffic": measured_traffic(args.config, args.mode, n, nm) if world == 1 else None}
                           for nm, st, b in zip(stage_names, stages, stage_bytes)},
                "whole_build": {"algorithmic_bytes": whole_bytes,
                                "achieved_gbs": whole_bytes / (ms / 1000.0) / 1e9,
                                "frac": whole_bytes / (ms / 1000.0) / 1e9 / peak}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mode = "average" if args.mode in ("color_filter", "average") else args.mode
        rate, times = cpu_reference_rate(kind, seed, args.cpu_sample, mode, steps=2)
        cpu = {"value": rate, "unit": "points/s", "cores": 1, "kind": "port",
               "sample": f"first {args.cpu_sample} points of {args.config}, {mode}, numpy oracle port of "
                         f"lodforge partition + build_lod (single-threaded like the reference), median of 2"}

    if rank == 0:
        line = {
            "metric": f"LOD construction points/sec ({args.mode})",
            "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64-geometry/u32-counts", "data": "synthetic",
            "config": {"workload": args.config, "points_per_gpu": n, "mode": args.mode, "T": 50_000,
                       "grid": 128, "l2": "input 16 B/pt x points > 126 MB L2, no flush",
                       "parallelism": f"subtree-sharded x{world} ({args.backend} all-reduce + all-to-all + rank-0 merge)"
                       if world > 1 else "single"},
            "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
            "stages_ms": dict(zip(stage_names, stages)),
            "tree": {"nodes": info.n_nodes, "leaves": info.n_leaves, "depth": info.depth, "voxels": V,
                     "ext_grids": info.n_ext_grids, "radix_passes": info.radix_passes},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
