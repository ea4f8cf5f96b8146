"""Degenerate / maximum-size shapes vs the oracle: python tools/edge_probe.py"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2004_10856_b200 as ft  # noqa: E402
from synth.graphs import Workload  # noqa: E402


def chain(K, seed=0, hi=1 << 30):
    rng = np.random.default_rng(seed)
    n = len(K)
    src = np.arange(n - 1, dtype=np.int32)
    dst = np.arange(1, n, dtype=np.int32)
    op_m = [rng.integers(0, hi, k).astype(np.int64) for k in K]
    op_t = [rng.integers(0, hi, k).astype(np.int64) for k in K]
    edge_t = [rng.integers(0, hi, K[i] * K[i + 1]).astype(np.int64) for i in range(n - 1)]
    return Workload(f"chain{K}", np.array(K, np.int32), src, dst, op_m, op_t, edge_t).check()


for K in ([1], [7], [4096], [4096, 4096], [2000, 3000], [1, 4096, 1], [4096, 1, 4096]):
    w = chain(K)
    t0 = time.time()
    og = oracle.load(w, 16)
    og.eliminate()
    om, ot = og.frontier()
    t1 = time.time()
    try:
        g = ft.load(w)
        g.eliminate()
        gm, gt = g.frontier()
        ok = np.array_equal(om, gm) and np.array_equal(ot, gt)
        print(K, "frontier", len(om), "match", ok, f"oracle {t1 - t0:.1f}s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(K, "GPU error:", e, flush=True)
