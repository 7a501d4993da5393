"""Last build's launch list (ncu csv with time + DRAM bytes): per-kernel totals."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    per.setdefault(int(r[0]), {"k": r[ki].split("(")[0][-44:]})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.items())
start = max(i for i, (_, d) in enumerate(items) if "k_bounds" in d["k"] and "finalize" not in d["k"])
agg = collections.OrderedDict()
tot = [0.0, 0.0, 0.0]
for _, d in items[start:]:
    t, rd, wr = d.get("gpu__time_duration.sum", 0) / 1e3, d.get("dram__bytes_read.sum", 0) / 1e6, d.get("dram__bytes_write.sum", 0) / 1e6
    a = agg.setdefault(d["k"], [0, 0.0, 0.0, 0.0])
    a[0] += 1; a[1] += t; a[2] += rd; a[3] += wr
    tot[0] += t; tot[1] += rd; tot[2] += wr
print(f"{'kernel':46s} {'n':>3s} {'us':>9s} {'rd MB':>9s} {'wr MB':>9s} {'GB/s':>7s}")
for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:46s} {n:3d} {t:9.1f} {rd:9.1f} {wr:9.1f} {(rd + wr) / t * 1e3 if t else 0:7.0f}")
print(f"{'total':46s} {len(items) - start:3d} {tot[0]:9.1f} {tot[1]:9.1f} {tot[2]:9.1f}")
