"""Per-wave breakdown of one search (profile events on)."""
import sys
sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402
name = sys.argv[1]
w = G.get(name)
for rep in range(2):
    g = ft.load(w, profile=True)
    g.prepare()
    g.eliminate()
    g.frontier()
st = g.stats()
waves = {}
for s in st:
    d = waves.setdefault(s["wave"], {"kinds": {}, "tuples": 0, "ms": 0.0, "launches": 0, "levels": 0,
                                      "filter": 0.0, "bucket": 0.0, "direct": 0.0, "cand": 0, "nseg": 0})
    d["kinds"][s["kind"]] = d["kinds"].get(s["kind"], 0) + 1
    d["tuples"] += s["tuples"]
    d["nseg"] += s["nseg"]
    d["ms"] += s["kernel_ms"]
    d["launches"] += s["launches"]
    d["levels"] = max(d["levels"], s["levels"])
    d["filter"] += s["filter_ms"]
    d["bucket"] += s["bucket_ms"]
    d["direct"] += s["direct_ms"]
    d["cand"] += s["candidates"]
tot = sum(d["ms"] for d in waves.values())
print(f"{name}: {len(waves)} waves, kernel ms {tot:.2f}")
for k in sorted(waves, key=lambda k: -waves[k]["ms"])[:25]:
    d = waves[k]
    print(f"wave {k:3d} {str(d['kinds']):38s} nseg {d['nseg']:8d} tuples {d['tuples']:12d} lev {d['levels']} "
          f"ms {d['ms']:7.3f} filt {d['filter']:6.3f} buck {d['bucket']:6.3f} dir {d['direct']:6.3f} cand {d['cand']:9d} launch {d['launches']}")
small = [d for d in waves.values() if d["ms"] < 0.5]
print(f"{len(small)} waves < 0.5 ms: total {sum(d['ms'] for d in small):.2f} ms")
