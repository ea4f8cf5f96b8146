"""Per-step-kind breakdown of one FT search (GPU).  Usage:
python tools/profile_run.py C4 [key=val ...]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402


def main():
    name = sys.argv[1]
    kw = {}
    for a in sys.argv[2:]:
        k, v = a.split("=")
        kw[k] = float(v) if "." in v else int(v)
    w = G.get(name, **kw)
    for rep in range(2):
        t0 = time.perf_counter()
        g = ft.load(w, profile=True)
        g.prepare()
        t1 = time.perf_counter()
        g.eliminate()
        m, t = g.frontier()
        t2 = time.perf_counter()
        st = g.stats()
    agg = {}
    for s in st:
        a = agg.setdefault(s["kind"], {"n": 0, "tuples": 0, "cand": 0, "surv": 0, "ms": 0.0,
                                       "plan": 0.0, "direct": 0.0, "filter": 0.0, "bucket": 0.0,
                                       "compact": 0.0, "maxlev": 0, "retries": 0, "launches": 0,
                                       "max_tuples": 0, "host": 0.0, "max_seg": 0})
        a["n"] += 1
        a["tuples"] += s["tuples"]
        a["max_tuples"] = max(a["max_tuples"], s["tuples"])
        a["cand"] += s["candidates"]
        a["surv"] += s["survivors"]
        a["ms"] += s["kernel_ms"]
        a["max_seg"] = max(a["max_seg"], s["max_seg"])
        for k in ("plan", "direct", "filter", "bucket", "compact", "host"):
            a[k] += s[k + "_ms"]
        a["maxlev"] = max(a["maxlev"], s["levels"])
        a["retries"] += s["retries"]
        a["launches"] += s["launches"]
    tot_t = sum(a["tuples"] for a in agg.values())
    tot_ms = sum(a["ms"] for a in agg.values())
    print(json.dumps({"workload": w.name, "steps": len(st), "frontier": len(m),
                      "tuples": tot_t, "kernel_ms": round(tot_ms, 3), "wall_ms": round((t2 - t1) * 1e3, 3),
                      "prepare_ms": round((t1 - t0) * 1e3, 3),
                      "Gtuples_per_s_kernel": round(tot_t / tot_ms / 1e6, 3)}))
    for k, a in agg.items():
        print(k, json.dumps({kk: (round(v, 3) if isinstance(v, float) else v) for kk, v in a.items()}))
    top = sorted(st, key=lambda s: -s["kernel_ms"])[:int(kw.pop("top", 3)) if False else 3]
    for s in top:
        print("top", json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()}))


if __name__ == "__main__":
    main()
