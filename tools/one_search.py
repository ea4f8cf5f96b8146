"""One FT search of a workload on cuda:0 (for ncu).  With --target KERNEL,
prints the ncu launch-skip count that lands on KERNEL's level-0 launch in the
wave with the largest work for that kernel family:
  k_filter / k_bucket_small: launched once per filter level (levels-1 per wave)
  k_direct_warp / k_direct:  launched once per level (levels per wave)"""
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
    kern = sys.argv[sys.argv.index("--target") + 1]
    waves = {}
    for s in st:
        waves.setdefault(s["wave"], s)  # first step of each wave carries the wave numbers
    order = [waves[w] for w in sorted(waves)]
    per = (lambda s: max(0, s["levels"] - 1)) if kern in ("k_filter", "k_bucket_small") else (lambda s: s["levels"])
    key = "filter_tuples" if kern in ("k_filter", "k_bucket_small") else "direct_tuples"
    best = max(range(len(order)), key=lambda i: order[i][key])
    if "--wave" in sys.argv:
        best = int(sys.argv[sys.argv.index("--wave") + 1])
    skip = sum(per(s) for s in order[:best]) + max(0, per(order[best]) - 1)
    print(f"target {kern} wave {best} {key} {order[best][key]} levels {order[best]['levels']} skip {skip}")
print("frontier", len(m))
