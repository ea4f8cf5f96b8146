"""Run named test functions of tests/test_gpu_parity.py in order, then the
wide [4096,4096] shape; print PASS/FAIL.  python tools/bisect_prelude.py name[:arg] ..."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2004_10856_b200 as ft  # noqa: E402
import test_gpu_parity as T  # noqa: E402

for spec in sys.argv[1:]:
    name, _, arg = spec.partition(":")
    fn = getattr(T, name)
    if arg:
        fn(ft, int(arg))
    elif name == "test_shared_path_ab":
        fn(ft, None)
    else:
        fn(ft)
import numpy as np  # noqa: E402
import oracle  # noqa: E402
w = T._wide([4096, 4096], [(0, 1)])
og = oracle.load(w, 16)
og.eliminate()
og.frontier()
g = ft.load(w, keep_all=True)
g.eliminate()
g.frontier()
so, m, t, bp = g.step_output(0)
oso, om, ot, obp = og.step_output(0)
gc, oc = np.diff(so), np.diff(oso)
bad = np.nonzero(gc != oc)[0]
print("PASS" if len(bad) == 0 else "FAIL", sys.argv[1:], "bad segs", len(bad), "first", bad[:6].tolist(),
      "gpu cnt", gc[bad[:6]].tolist(), "oracle cnt", oc[bad[:6]].tolist(), "gpu total", int(gc.sum()),
      "oracle total", int(oc.sum()), "zero segs", int((gc == 0).sum()))
if len(bad):
    s0 = int(bad[0])
    print(" seg", s0, "gpu m", m[so[s0]:so[s0 + 1]][:5].tolist(), "oracle m", om[oso[s0]:oso[s0 + 1]][:5].tolist())
