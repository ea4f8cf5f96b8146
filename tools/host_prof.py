"""Host-side phase times of warm searches (FT_HOST_PROF=1 prints them when a
graph is destroyed): python tools/host_prof.py C5 [repeats]"""
import os
import sys

os.environ["FT_HOST_PROF"] = "1"
sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

w = G.get(sys.argv[1] if len(sys.argv) > 1 else "C5")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    g = ft.load(w)
    g.prepare()
    g.eliminate()
    g.frontier()
    g.close()
