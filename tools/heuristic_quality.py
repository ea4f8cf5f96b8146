"""S:603 (acceptance criterion 3) report: on 50 shared-input fixtures
(synth.random_masked: a K>=2 mask-like source feeding several ops), run the
oracle's FT_AUTO_HEUR with each configuration rule and report the mean
fraction of the exact (brute-force) frontier that the heuristic output
weakly dominates, plus how many fixtures lost points.  CPU only.

    python tools/heuristic_quality.py [--out profiles/r2_heuristic_quality.json]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import bruteforce as bf  # noqa: E402
from synth import graphs as G  # noqa: E402


def run(policy, alpha):
    fr, lossy, n = [], 0, 0
    for seed in range(50):
        w = G.random_masked(1000 + seed, n_ops=4 + seed % 3, kmax=3, mask_k=3, fanout=3, cost_hi=40)
        g = oracle.load(w, 2)
        g.set_heuristic(policy, alpha)
        g.eliminate(oracle.AUTO_HEUR)
        try:
            m, t = g.frontier()
        except oracle.OracleError:
            continue
        n += 1
        ex = bf.brute_force(w)
        f = sum(bool(((m <= a) & (t <= b)).any()) for a, b in ex) / len(ex)
        fr.append(f)
        lossy += f < 1.0
    return {"policy": policy, "alpha": list(alpha) if policy == "weighted" else None, "fixtures": n,
            "mean_fraction_dominated": float(np.mean(fr)), "min_fraction": float(np.min(fr)),
            "fixtures_with_loss": int(lossy)}


def main():
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    rows = [run("min_memory", (1, 1))] + [run("weighted", a) for a in ((1, 2), (1, 4), (3, 4), (0, 1))]
    for r in rows:
        print(json.dumps(r))
    if out:
        json.dump({"criterion": "SPEC S:603 acceptance criterion 3", "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
