"""Summarise an ncu report: key throughput metrics + top SASS stall reasons per kernel.

    python scripts/ncu_summary.py gpurun_out/prof_k_radix.ncu-rep [--sass N]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size"]
STALLS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_drain", "stall_lg", "stall_long_sb",
          "stall_math", "stall_membar", "stall_mio", "stall_misc", "stall_no_inst", "stall_not_selected",
          "stall_selected", "stall_short_sb", "stall_sleep", "stall_tex", "stall_wait"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    h = rows[0]
    units = rows[1]
    out = []
    for r in rows[2:]:
        d = {"name": r[h.index("Kernel Name")][:70], "id": r[0]}
        for k in KEYS:
            if k in h:
                d[k] = (r[h.index(k)], units[h.index(k)])
        out.append(d)
    return out


def sass(rep, top):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    res = []
    for b in blocks:
        if not b["rows"]:
            continue
        h = b["rows"][0]
        si = h.index("Warp Stall Sampling (All Samples)")
        data = [r for r in b["rows"][1:] if len(r) > si and r[si] not in ("", "0")]
        tot = sum(float(r[si]) for r in data) or 1
        agg = {}
        for st in STALLS:
            if st in h:
                agg[st] = sum(float(r[h.index(st)] or 0) for r in data) / tot * 100
        hot = sorted(data, key=lambda r: -float(r[si]))[:top]
        res.append((b["name"][:60], agg, [(float(r[si]) / tot * 100, r[h.index("Source")].strip()[:90]) for r in hot]))
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 12
    for d in raw(rep):
        print(f"== [{d['id']}] {d['name']}")
        for k in KEYS:
            if k in d:
                print(f"   {k:62s} {d[k][0]:>16s} {d[k][1]}")
    for name, agg, hot in sass(rep, top):
        print(f"-- stalls {name}: " + ", ".join(f"{k[6:]}={v:.0f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]))
        for pct, src in hot:
            print(f"   {pct:5.1f}%  {src}")
