"""Generate golden digests by running the REAL reference (`lodforge`, /root/reference).

Build-container only (the reference does not travel to the GPU box):

    python tests/golden/make_golden.py [--quick] [name ...]

For every case in `cases.py` it
  1. regenerates the input with the reference's own `generate` (reference
     presets) and asserts our restated generator is byte-identical;
  2. runs `lodforge.partition.partition` + `lodforge.sampling.build_lod` for each
     mode, unmodified;
  3. writes tests/golden/<name>.json.gz: per-node digests in the format of
     `oracle/lod_oracle.split_digest` / `voxel_digest`, or the exception text
     when the reference raises (e.g. the 2^20 random-sampling limit).  "weighted" stores
     sha1(coords) and the zlib+base64 colours (compared within +-1 per channel);
  4. records [length, sha1] of the reference's VLPC file (codec.encode) per mode.
"""
from __future__ import annotations

import base64
import gzip
import io
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import zlib  # noqa: E402

import numpy as np  # noqa: E402

import cases as C  # noqa: E402


def _sha(*arrays):
    h = hashlib.sha1()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _ps(path):
    return "".join(str(o) for o in path) or "-"


def run_case(case):
    from lodforge.codec import encode
    from lodforge.errors import ConsistencyError
    from lodforge.ingest import GeneratorPreset, PointCloud, generate
    from lodforge.model import BuildConfig
    from lodforge.partition import partition
    from lodforge.sampling import build_lod

    t0 = time.time()
    pos, col = C.make_input(case)
    spec = case["spec"]
    if spec[0] == "ref":
        ref = generate(GeneratorPreset(spec[1], spec[2], spec[3]))
        assert np.array_equal(ref.positions, pos), case["name"]
        if case.get("color") is None:
            assert np.array_equal(ref.colors, col), case["name"]
    cloud = PointCloud(np.asarray(pos, np.float64), col)
    cfg = BuildConfig(**case["cfg"])
    out = {"name": case["name"], "n": len(cloud), "input_sha": _sha(cloud.positions, cloud.colors)}
    tree = partition(cloud, cfg)
    split = {}
    for nd in tree.iter_nodes():
        b = [float(v).hex() for v in nd.bounds.min] + [float(nd.bounds.size).hex()]
        if nd.is_leaf:
            split[_ps(nd.path)] = ["L", nd.point_count, bool(nd.oversized), b,
                                   _sha(nd.point_positions, nd.point_colors)]
        else:
            split[_ps(nd.path)] = ["I", 0, False, b, ""]
    out["world"] = [float(v).hex() for v in tree.world_bounds.min] + [float(tree.world_bounds.size).hex()]
    out["split"] = split
    modes, vlpc = {}, {}
    for mode in case["modes"]:
        strat, _, seed = mode.partition(":")
        try:
            build_lod(tree, strat, int(seed or 0))
            if strat != "weighted":   # the file of `lodforge build --strategy S --seed K` (cli.py:98-118)
                tree.config.strategy, tree.config.seed = strat, int(seed or 0)
                buf = io.BytesIO()
                encode(tree, buf)
                vlpc[mode] = [len(buf.getvalue()), hashlib.sha1(buf.getvalue()).hexdigest()]
            if strat == "weighted":   # +-1 tolerance: keep the colours themselves
                modes[mode] = {_ps(nd.path): [nd.voxel_count, _sha(nd.voxel_coords),
                                              base64.b64encode(zlib.compress(
                                                  np.ascontiguousarray(nd.voxel_colors, np.uint8).tobytes(), 9)
                                              ).decode()]
                               for nd in tree.inner_nodes()}
            else:
                modes[mode] = {_ps(nd.path): [nd.voxel_count, _sha(nd.voxel_coords, nd.voxel_colors)]
                               for nd in tree.inner_nodes()}
        except ConsistencyError as e:
            modes[mode] = {"error": str(e)}
    out["modes"] = modes
    out["vlpc"] = vlpc
    out["seconds"] = round(time.time() - t0, 2)
    with gzip.open(os.path.join(HERE, case["name"] + ".json.gz"), "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    return case["name"], out["seconds"], len(split)


def main(argv):
    quick = "--quick" in argv
    names = [a for a in argv if not a.startswith("--")]
    todo = [c for c in C.CASES if (not names or c["name"] in names) and (c["quick"] or not quick)]
    todo.sort(key=lambda c: -len(c["name"]) if c["quick"] else -1_000)
    with mp.get_context("fork").Pool(min(8, os.cpu_count() or 1), maxtasksperchild=1) as pool:
        for name, sec, nn in pool.imap_unordered(run_case, todo):
            print(f"{name}: {nn} nodes, {sec}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
