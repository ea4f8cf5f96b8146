"""Aggregate ncu warp-stall samples and executed instructions of one kernel
by CUDA source line (SASS offsets mapped with nvdisasm -g).

usage: python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTR [top]"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
# a report with several launches prints one block per launch: summed by SASS offset
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
    elif r and r[0] != "Address" and cur is not None:
        cur.append(r)
d = [[None] * len(h) for _ in range(max(len(b) for b in blocks))]
for b in blocks:
    for i, r in enumerate(b):
        for c in (h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")):
            d[i][c] = str(float(d[i][c] or 0) + float(r[c] or 0))
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
# offset -> source line
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines = {}
for cub in glob.glob(tmp + "/*.cubin"):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    sec, cur = None, "?"
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            sec = ln
            continue
        if sec is None or kern not in sec:
            continue
        m = re.search(r'line (\d+)', ln)
        if "## File" in ln and m:
            f = re.search(r'File "([^"]+)"', ln)
            cur = f"{os.path.basename(f.group(1)) if f else '?'}:{m.group(1)}"
            continue
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
        if m:
            lines[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0.0, 0.0])
ts = te = 0.0
for i, r in enumerate(d):
    s, e = float(r[iss] or 0), float(r[iex] or 0)
    ts += s
    te += e
    k = lines.get(i * 16, "?")
    agg[k][0] += s
    agg[k][1] += e
for k, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{k:28s} stall {100*s/ts:5.1f}%  inst {100*e/te:5.1f}%")
