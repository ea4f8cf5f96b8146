"""Host-side phases of the end-to-end path (graph create, cost upload,
eliminate, frontier, close) on cuda:0: python tools/e2e_probe.py [C5]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

w = G.get(sys.argv[1] if len(sys.argv) > 1 else "C5")
pinned = []
for a in ft.concat_costs(w):
    if a is None:
        pinned.append(None)
        continue
    pt = torch.empty(len(a), dtype=torch.int64, pin_memory=True)
    pt.numpy()[:] = a
    pinned.append(pt.numpy())
g = ft.load(w)
g.eliminate()
g.frontier()
g.close()
for i in range(6):
    sync = torch.cuda.synchronize
    sync()
    t0 = time.perf_counter()
    g = ft.Graph(w.n_cfgs, w.src, w.dst)
    sync()
    t1 = time.perf_counter()
    g.set_costs_all(*pinned)
    sync()
    t2 = time.perf_counter()
    g.prepare()
    sync()
    t3 = time.perf_counter()
    g.eliminate()
    sync()
    t4 = time.perf_counter()
    g.frontier()
    sync()
    t5 = time.perf_counter()
    g.close()
    sync()
    t6 = time.perf_counter()
    print(i, "create %.2f costs %.2f prepare %.2f elim %.2f front %.2f close %.2f" %
          tuple((b - a) * 1e3 for a, b in ((t0, t1), (t1, t2), (t2, t3), (t3, t4), (t4, t5), (t5, t6))))
