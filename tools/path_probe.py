"""Kernel-path counters (ft_step_stats.path) summed over a search, per workload."""
import sys

sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

cases = {
    "c5_small": lambda: G.c5(seed=3, n_ops=60, K=16),
    "c5_k64": lambda: G.c5(seed=3, n_ops=40, K=64),
    "sp_ties": lambda: G.random_sp(7, n_ops=30, kmax=24, cost_hi=4),
    "sp_wide": lambda: G.random_sp(8, n_ops=30, kmax=32, cost_hi=1 << 20),
    "c4_l2": lambda: G.c4(layers=2),
    "c3": lambda: G.c3(),
}
for name, mk in cases.items():
    w = mk()
    g = ft.load(w)
    g.eliminate()
    tot = {}
    for s in g.stats():
        for k, v in s["path"].items():
            tot[k] = tot.get(k, 0) + v
    print(name, tot, flush=True)
