"""Loopback virtual ranks on one GPU vs world 1: first differing steps.

usage: python tools/loop_check.py WORKLOAD WORLD"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

name, world = sys.argv[1], int(sys.argv[2])
w = G.get(name)
a = ft.load(w, keep_all=True)
a.eliminate()
b = ft.load(w, keep_all=True, world=world, loopback=1)
b.eliminate()
sa, sb = a.stats(), b.stats()
bad = []
for s in range(len(sa)):
    x, y = a.step_output(s), b.step_output(s)
    if not all(np.array_equal(u, v) for u, v in zip(x, y)):
        bad.append(s)
print(name, "world", world, "bad steps", len(bad), bad[:10])
for s in bad[:4]:
    (so, m, t, bp), (so2, m2, t2, bp2) = a.step_output(s), b.step_output(s)
    seg = np.nonzero(np.diff(so) != np.diff(so2))[0] if len(so) == len(so2) else "nseg"
    print(" step", s, sa[s]["kind"], "wave", sa[s]["wave"], "nseg", sa[s]["nseg"], "nblk", sa[s]["nblk"],
          "levels", sa[s]["levels"], "diff segs", seg[:8] if not isinstance(seg, str) else seg,
          "n", len(m), len(m2))
