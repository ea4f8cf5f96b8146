"""Map SASS byte offsets of one kernel to CUDA source lines (nvdisasm -g).

usage: python tools/sass_lines.py LIB.so KERNEL_SUBSTR OFF [OFF ...]   (decimal offsets, as ncu prints)"""
import glob
import os
import re
import subprocess
import sys
import tempfile

lib, kern, offs = sys.argv[1], sys.argv[2], [int(x) for x in sys.argv[3:]]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
for cub in glob.glob(d + "/*.cubin"):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    sec = None
    line = ""
    found = {}
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            sec = ln
            continue
        if sec is None or kern not in sec:
            continue
        m = re.search(r'line (\d+)', ln)
        if "## File" in ln and m:
            f = re.search(r'File "([^"]+)"', ln)
            line = f"{os.path.basename(f.group(1)) if f else '?'}:{m.group(1)}"
            continue
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*)', ln)
        if m:
            o = int(m.group(1), 16)
            if any(abs(o - x) <= 32 for x in offs):
                found[o] = (line, m.group(2).strip()[:70])
    for o in sorted(found):
        print(f"{o:6d} {found[o][0]:28s} {found[o][1]}")
