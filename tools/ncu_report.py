"""Write profiles/<name>.md from an ncu launch-list CSV and full-set reports.

usage: python tools/ncu_report.py OUT.md LAUNCHES.csv REPORT.ncu-rep ...
"""
import collections
import csv
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import KEYS, hot, raw  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
        "ms": 1e6, "msecond": 1e6, "nsecond": 1}


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("ftk::", "")
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
        if r[mi] == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += v
        elif r[mi] == "dram__bytes_read.sum":
            agg[name][2] += v
        elif r[mi] == "dram__bytes_write.sum":
            agg[name][3] += v
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | ms (serialised, cold) | share | DRAM read GB | DRAM write GB |",
           "|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {a[0]} | {a[1] / 1e6:.3f} | {a[1] / tot:.3f} | {a[2] / 1e9:.3f} | {a[3] / 1e9:.3f} |")
    out.append(f"| total | {sum(a[0] for a in agg.values())} | {tot / 1e6:.3f} | 1.000 | | |")
    return out


def main():
    out_md, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [f"# ncu summary ({os.path.basename(out_md)})", ""]
    if os.path.exists(launches):
        lines += [f"## Launch list: `{os.path.basename(launches)}`", "",
                  "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none` (per-launch times are cold-cache and serialised: compare shares).",
                  ""] + launch_table(launches) + [""]
    for rep in reps:
        m = raw(rep)
        lines += [f"## Full set: `{os.path.basename(rep)}`", "", "| metric | value |", "|---|---|"]
        for k in KEYS:
            if k in m:
                lines.append(f"| {k} | {m[k][0]} {m[k][1]} |")
        lines += ["", "Hottest SASS windows (24 instructions; share of stall samples / executed instructions):", ""]
        for s, e, i, src in hot(rep):
            lines.append(f"- sass[{i}:] stall {s:.3f} inst {e:.3f} `{src}`")
        lines.append("")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print(out_md)


if __name__ == "__main__":
    main()
