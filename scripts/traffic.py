"""Per-stage DRAM traffic of one build from an ncu launch list (metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum) -> profiles/traffic.json[<config>:<mode>].

    python scripts/traffic.py gpurun_out/launches.csv terrain20M color_filter 20000000

Stages follow the library's stage events (api.cu mark()): bounds+count | extension |
merge+nodes+targets | distribute | voxelize, split at the first kernel of each stage."""
import collections
import csv
import json
import os
import sys

path, config, mode, points = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    per.setdefault(int(r[0]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.values())
start = max(i for i, d in enumerate(items) if "k_bounds" in d["k"] and "finalize" not in d["k"])
stage, out = 0, collections.OrderedDict((s, 0.0) for s in
                                       ["bounds+count", "extension", "merge+nodes+targets", "distribute", "voxelize"])
names = list(out)
for d in items[start:]:
    k = d["k"]
    # (the candidate-cell compaction, CandF, runs inside the count stage)
    if stage == 0 and (("k_compact" in k and "CandF" not in k) or "k_ext" in k or "k_mark_anchors" in k or "k_merge" in k):
        stage = 1
    if stage <= 1 and ("k_mark_anchors" in k or "k_merge" in k):
        stage = 2
    if stage <= 2 and ("k_digit_hist" in k or "k_dist_" in k):
        stage = 3
    if stage <= 3 and "k_setup" in k:
        stage = 4
    b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    out[names[stage]] += b
    if "k_dist_scatter" in k:   # the dominant single kernel (bench.py roofline)
        out["k_dist_scatter"] = out.get("k_dist_scatter", 0.0) + b
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
t = json.load(open(dst)) if os.path.exists(dst) else {}
t[f"{config}:{mode}"] = {"points": points, "stages": {k: int(v) for k, v in out.items()},
                         "source": os.path.basename(path)}
json.dump(t, open(dst, "w"), indent=1)
print(json.dumps(t[f"{config}:{mode}"]))
