"""One FT search of a workload on cuda:0 (for ncu); prints the k_filter
launch index of the largest step (ncu --launch-skip target) when --target."""
import sys

sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
g = ft.load(G.get(name))
g.eliminate()
m, t = g.frontier()
st = g.stats()
if "--target" in sys.argv:
    best = max(range(len(st)), key=lambda i: st[i]["tuples"])
    skip = sum(max(0, s["levels"] - 1) for s in st[:best]) + max(0, st[best]["levels"] - 2)
    print(f"largest step {best} tuples {st[best]['tuples']} levels {st[best]['levels']} filter_skip {skip}")
print("frontier", len(m))
