"""Per-kernel totals from ncu launch-list CSVs: python tools/kern_totals.py A.csv [B.csv ...]"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        n = r[ki].split("(")[0].replace("void ", "")
        agg[n][0] += 1
        agg[n][1] += float(r[vi].replace(",", "")) / 1e6
    tot = sum(v[1] for v in agg.values())
    print(path, "total ms", round(tot, 2), "launches", sum(v[0] for v in agg.values()))
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"  {n:28s} {c:6d} {t:8.2f}")
