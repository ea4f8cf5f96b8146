"""Warm host-side profile of the library (FT_HOST_PROF): python tools/host_prof.py C4"""
import os
import sys
import time

os.environ["FT_HOST_PROF"] = "1"
sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

w = G.get(sys.argv[1] if len(sys.argv) > 1 else "C4")
for i in range(3):
    g = ft.load(w)
    g.prepare()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.eliminate()
    g.frontier()
    torch.cuda.synchronize()
    print(f"search {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms wall", file=sys.stderr, flush=True)
    g.close()
