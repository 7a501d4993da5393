"""Print the last build's kernel launch list from gpurun_out/launches.csv (ncu) with totals."""
import csv, sys, collections
path = sys.argv[1] if len(sys.argv) > 1 else "/root/repo/gpurun_out/launches.csv"
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
items = [(int(r[ii]), r[ki].split("(")[0][-40:], float(r[vi].replace(",", "")) / 1000) for r in data]
# the last build starts at the last k_bounds launch
start = max(i for i, (_, k, _) in enumerate(items) if "k_bounds<" in k)
last = items[start:]
agg = collections.OrderedDict()
for i, k, v in last:
    if v >= thr: print(f"{i:5d} {v:9.1f} us  {k}")
    agg[k] = agg.get(k, 0) + v
print("---- per kernel (us):", ", ".join(f"{k.split('::')[-1]}={v:.0f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]))
print(f"total {sum(v for *_, v in last):.1f} us over {len(last)} launches")
