"""Per-kernel (and per kernel-group) totals of ONE FT search from an ncu
launch list, for bench.py's roofline (profiles/r2_kernels.json).

    ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,\
dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,\
smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
        --log-file L.csv python tools/one_search.py C5
    python tools/kernel_table.py L.csv C5 [--out profiles/r2_kernels.json]

Times are serialised, cold-cache ncu times (compare SHARES with the live
CUDA-event split); instruction and DRAM byte counts are properties of the
workload (deterministic up to atomics' ordering)."""
import collections
import csv
import json
import os
import re
import sys

GROUP = {"k_filter": "filter", "k_direct_warp": "direct", "k_direct": "direct", "k_node_pack": "direct",
         "k_node_shared": "direct", "k_carry": "bucket", "k_scatter": "bucket", "k_bucket_small": "bucket",
         "k_bucket_large": "bucket", "k_plan": "plan"}


def base(name):
    n = re.sub(r"^void\s+", "", name)
    n = n.split("(")[0].split("<")[0]
    return n.replace("ftk::", "").strip()


def table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "") or 0)
        names[r[ii]] = base(r[ki])
    agg = collections.defaultdict(lambda: collections.Counter())
    for lid, m in per.items():
        k = names[lid]
        a = agg[k]
        a["launches"] += 1
        t = m.get("gpu__time_duration.sum", 0.0)
        a["time_ns"] += t
        a["inst"] += m.get("smsp__inst_executed.sum", 0.0)
        a["dram"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["sm_pct_t"] += t * m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0.0)
        a["issue_pct_t"] += t * m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0)
    return agg


def entry(a):
    t = a["time_ns"] or 1.0
    return {"launches_per_search": int(a["launches"]), "ncu_ms_per_search": a["time_ns"] / 1e6,
            "inst_per_search": a["inst"], "dram_bytes_per_search": a["dram"],
            "sm_throughput_pct": a["sm_pct_t"] / t, "issue_active_pct": a["issue_pct_t"] / t}


def main():
    path, workload = sys.argv[1], sys.argv[2]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    agg = table(path)
    kernels = {k: entry(a) for k, a in agg.items()}
    groups = collections.defaultdict(collections.Counter)
    for k, a in agg.items():
        groups[GROUP.get(k, "compact")].update(a)
    tot = sum(a["time_ns"] for a in agg.values())
    res = {"source": f"ncu launch list of tools/one_search.py {workload} ({os.path.basename(path)})",
           "total_ncu_ms": tot / 1e6, "launches": int(sum(a["launches"] for a in agg.values())),
           "kernels": dict(kernels, **{g: entry(a) for g, a in groups.items()})}
    for k, e in sorted(kernels.items(), key=lambda x: -x[1]["ncu_ms_per_search"]):
        print(f"{k:18s} {e['launches_per_search']:6d} {e['ncu_ms_per_search']:9.3f} ms "
              f"{100 * e['ncu_ms_per_search'] * 1e6 / tot:5.1f}%  inst {e['inst_per_search']:.3e}  "
              f"dram {e['dram_bytes_per_search'] / 1e6:9.1f} MB  sm {e['sm_throughput_pct']:5.1f}%  "
              f"issue {e['issue_active_pct']:5.1f}%")
    if out:
        d = json.load(open(out)) if os.path.exists(out) else {}
        d[workload] = res
        json.dump(d, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
