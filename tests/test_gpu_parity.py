"""GPU parity: libft (CUDA, sm_100a) vs the CPU oracle, element by element.

Every step's output set (seg_off, m, t, bp) must be bit-identical to the
oracle's (integer work: exact), as must the final frontier and every
unrolled strategy (SURVEY 8(c) "GPU <-> oracle")."""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
from synth import graphs as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ft():
    import paper_2004_10856_b200 as ft
    return ft


def compare(ft, w, threads=8, strategies="all", stride=1):
    og = oracle.load(w, threads)
    og.eliminate()
    om, ot = og.frontier()
    gg = ft.load(w, keep_all=True)
    gg.eliminate()
    gm, gt = gg.frontier()
    st = gg.stats()
    assert og.num_steps() == len(st)
    for s in range(0, len(st), stride):
        info = og.step_info(s)
        assert info["kind"] == st[s]["kind"], s
        assert info["tuples"] == st[s]["tuples"], s
        a = og.step_output(s)
        b = gg.step_output(s)
        for name, x, y in zip(("seg_off", "m", "t", "bp"), a, b):
            if not np.array_equal(x, y):
                bad = np.nonzero(x != y)[0][:5] if len(x) == len(y) else "len"
                raise AssertionError(f"{w.name} step {s} ({info['kind']}) {name} differs at {bad}")
    assert np.array_equal(om, gm) and np.array_equal(ot, gt)
    idx = range(len(om)) if strategies == "all" else np.linspace(0, len(om) - 1, strategies).astype(int)
    for i in idx:
        assert np.array_equal(og.strategy(int(i)), gg.strategy(int(i))), i
    return gg, st


def test_c1_seeds(ft):
    for seed in range(100):
        for var in ("chain", "parallel", "diamond"):
            compare(ft, G.c1(seed, var))


def test_random_sp(ft):
    for seed in range(200):
        w = G.random_sp(seed, n_ops=2 + seed % 12, kmax=4, edge_mem=(seed % 5 == 0))
        compare(ft, w)


def test_random_sp_large_frontiers(ft):
    """Wider cost ranges and K: multi-level (filter) path with ragged segments."""
    for seed in range(12):
        w = G.random_sp(1000 + seed, n_ops=14, kmax=12, cost_hi=1 << 20)
        compare(ft, w)


def test_c2_vgg(ft):
    compare(ft, G.c2())


def test_c2_no_jitter_ties(ft):
    compare(ft, G.c2(jitter=False))


def test_c3_resnet(ft):
    gg, st = compare(ft, G.c3(), strategies=64)
    assert max(s["levels"] for s in st) >= 2  # the filter path ran


def test_c4_bert_2layers(ft):
    compare(ft, G.c4(layers=2), strategies=32)


def test_c5_small(ft):
    compare(ft, G.c5(n_ops=200, K=16, B=8, Lmin=2, Lmax=6), strategies=32)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_invariance_loopback(ft, world):
    """Multi-rank sharding (virtual ranks on one GPU): every step output and the
    strategies are bit-identical to world = 1 (ids are shard-invariant, R6)."""
    for w in (G.c3(), G.c4(layers=2), G.c5(n_ops=200, K=16, B=8, Lmin=2, Lmax=6)):
        a = ft.load(w, keep_all=True)
        a.eliminate()
        am, at = a.frontier()
        b = ft.load(w, keep_all=True, world=world, loopback=True)
        b.eliminate()
        bm, bt = b.frontier()
        assert np.array_equal(am, bm) and np.array_equal(at, bt)
        for s in range(len(a.stats())):
            for x, y in zip(a.step_output(s), b.step_output(s)):
                assert np.array_equal(x, y), (w.name, s)
        for i in np.linspace(0, len(am) - 1, 16).astype(int):
            assert np.array_equal(a.strategy(int(i)), b.strategy(int(i)))


def test_bert_no_jitter_ties(ft):
    """Exact m/t ties (no cost jitter): shared-order node path's tie rule."""
    compare(ft, G.c4(layers=3, jitter=False), strategies=16)


def test_shared_path_ab(ft, monkeypatch):
    """Shared-order node path vs the generic pipeline (FT_NO_SHARED): identical."""
    import os
    w = G.c5(n_ops=300, K=32, B=8, Lmin=3, Lmax=8)
    a = ft.load(w, keep_all=True)
    a.eliminate()
    am, at = a.frontier()
    os.environ["FT_NO_SHARED"] = "1"
    try:
        b = ft.load(w, keep_all=True)
        b.eliminate()
        bm, bt = b.frontier()
    finally:
        del os.environ["FT_NO_SHARED"]
    assert np.array_equal(am, bm) and np.array_equal(at, bt)
    for s in range(len(a.stats())):
        for x, y in zip(a.step_output(s), b.step_output(s)):
            assert np.array_equal(x, y), s


def test_bulk_vs_per_op_setters(ft):
    """ft_set_costs_all (device-validated bulk upload) == per-op/per-edge setters."""
    w = G.c3()
    a = ft.load(w, bulk=True)
    a.eliminate()
    b = ft.load(w, bulk=False)
    b.eliminate()
    for x, y in zip(a.frontier(), b.frontier()):
        assert np.array_equal(x, y)


def test_bulk_validation_errors(ft):
    w = G.c1(0)
    op_m, op_t, em, et = ft.concat_costs(w)
    for bad, code in (((-1), ft.EINVAL), ((1 << 40), ft.EOVERFLOW)):
        g = ft.Graph(w.n_cfgs, w.src, w.dst)
        et2 = et.copy()
        et2[3] = bad
        with pytest.raises(ft.FTError) as e:
            g.set_costs_all(op_m, op_t, em, et2)
        assert e.value.code == code
    g = ft.Graph(w.n_cfgs, w.src, w.dst)
    g.set_costs_all(op_m, op_t, em, et)
    with pytest.raises(ft.FTError) as e:
        g.set_op_costs(0, w.op_m[0], w.op_t[0])
    assert e.value.code == ft.ESTATE


def _paths(st):
    tot = {}
    for s in st:
        for k, v in s["path"].items():
            tot[k] = tot.get(k, 0) + v
    return tot


def test_kernel_paths_with_ties(ft):
    """Costs in [0, 4): heavy m ties.  Exercises every reduce path -- packed
    shared-order rows (k_node_pack), its equal-m group rule, the one-CTA-per-row
    fallback (k_node_shared) and the register-blocked CTA sort (k_direct) --
    and requires each to be bit-exact against the oracle."""
    tot = {}
    for seed in (7, 11, 19):
        _, st = compare(ft, G.random_sp(seed, n_ops=30, kmax=24, cost_hi=4), strategies=16)
        for k, v in _paths(st).items():
            tot[k] = tot.get(k, 0) + v
    assert tot["shared_rows"] > 0 and tot["shared_tie_rows"] > 0
    assert tot["shared_cta_rows"] > 0 and tot["direct_reg_segs"] > 0


def test_kernel_paths_wide_costs(ft):
    """Wide cost range (few ties): large shared rows (> 256 tuples, CTA
    fallback) and register-blocked direct segments without the tie rule."""
    tot = {}
    for seed in (8, 9):
        _, st = compare(ft, G.random_sp(seed, n_ops=30, kmax=32, cost_hi=1 << 20), strategies=16)
        for k, v in _paths(st).items():
            tot[k] = tot.get(k, 0) + v
    assert tot["shared_rows"] > 0 and tot["shared_cta_rows"] > 0 and tot["direct_reg_segs"] > 0


_PACK_REUSE = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2004_10856_b200 as ft
from synth import graphs as G
w = G.c5(n_ops=200, K=16, B=8, Lmin=2, Lmax=6)
a = ft.load(w, keep_all=True); a.eliminate()
bad = 0
for world in (2, 3):
    b = ft.load(w, keep_all=True, world=world, loopback=True); b.eliminate()
    for s in range(len(a.stats())):
        if not all(np.array_equal(x, y) for x, y in zip(a.step_output(s), b.step_output(s))):
            bad += 1
rows = sum(s["path"]["shared_rows"] for s in a.stats())
print("BAD", bad, "ROWS", rows)
"""


def test_partition_invariance_pack_reuse():
    """Rank boundaries cut shared-order rows into partial p ranges; with few
    k_node_pack CTAs (FT_PACK_GRID) each CTA reuses its staged t_z table across
    packs, which must be re-staged when the p range changes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FT_PACK_GRID="3")
    out = subprocess.run([sys.executable, "-c", _PACK_REUSE.format(root=root)], env=env, cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    tok = out.stdout.split()
    assert int(tok[tok.index("ROWS") + 1]) > 0
    assert int(tok[tok.index("BAD") + 1]) == 0, out.stdout


_KNOBS = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import oracle
import paper_2004_10856_b200 as ft
from synth import graphs as G
bad = steps = 0
for w in (G.c3(), G.c4(layers=2), G.c5(n_ops=300, K=32, B=8, Lmin=3, Lmax=8)):
    og = oracle.load(w, 8); og.eliminate(); om, ot = og.frontier()
    gg = ft.load(w, keep_all=True); gg.eliminate(); gm, gt = gg.frontier()
    bad += not (np.array_equal(om, gm) and np.array_equal(ot, gt))
    for s in range(og.num_steps()):
        steps += 1
        bad += not all(np.array_equal(x, y) for x, y in zip(og.step_output(s), gg.step_output(s)))
print("BAD", bad, "STEPS", steps)
"""


@pytest.mark.parametrize("knobs", [{"FT_PDL": "0"}, {"FT_FENCE": "0", "FT_BLOCK_SKIP": "0"},
                                   {"FT_FILTER_GRID": "148", "FT_PDL": "1"}])
def test_pipeline_knobs(knobs):
    """The per-process pipeline switches (read once per device runner, hence a
    subprocess each): plain stream launches instead of programmatic dependent
    launch, the per-lane G gallop instead of the warp-cooperative lower bound
    and no block-level pre-filter, a small filter grid (grid-stride passes) --
    every step still bit-exact against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _KNOBS.format(root=root)], env=dict(os.environ, **knobs),
                         cwd=root, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    tok = out.stdout.split()
    assert int(tok[tok.index("STEPS") + 1]) > 50
    assert int(tok[tok.index("BAD") + 1]) == 0, out.stdout


def _wide(K, edges, seed=0, hi=1 << 30):
    """Explicit graph with the given configuration counts and edges."""
    from synth.graphs import Workload
    rng = np.random.default_rng(seed)
    src = np.array([a for a, _ in edges], np.int32)
    dst = np.array([b for _, b in edges], np.int32)
    op_m = [rng.integers(0, hi, k).astype(np.int64) for k in K]
    op_t = [rng.integers(0, hi, k).astype(np.int64) for k in K]
    edge_t = [rng.integers(0, hi, K[a] * K[b]).astype(np.int64) for a, b in edges]
    return Workload(f"wide{K}", np.array(K, np.int32), src, dst, op_m, op_t, edge_t).check()


@pytest.mark.parametrize("K,edges", [
    ([4096], []),                                   # final reduce over 4096 singleton blocks
    ([4096, 4096], [(0, 1)]),                       # LDP: 4096 segments x 4096 blocks
    ([2000, 3000], [(0, 1)]),
    ([1, 4096, 1], [(0, 1), (1, 2)]),
    ([64, 4096, 64], [(0, 1), (1, 2), (0, 2)]),     # node elimination over 4096 blocks
    ([300, 300], [(0, 1), (0, 1), (0, 1)]),         # parallel multi-edges (Eq. 5 merges)
    ([1, 1, 1], [(0, 1), (1, 2), (0, 2)]),          # K = 1 everywhere
])
def test_extreme_shapes(ft, K, edges):
    """K up to the documented maximum (4096) and degenerate graphs: segments
    with more union terms than the direct capacity take the empty-staircase
    level (k_plan) and are reduced exactly by the bucket sorts."""
    compare(ft, _wide(K, edges), strategies=8)


def compare_elim(ft, w, threads=8, strategies=16):
    """FT-Elimination: every step bit-identical to the oracle's, and
    the frontier equal to FT-LDP's (both exact)."""
    og = oracle.load(w, threads)
    og.eliminate()
    om, ot = og.frontier(algo="elim")
    gg = ft.load(w, keep_all=True)
    gg.eliminate()
    gm, gt = gg.frontier(algo="elim")
    st = gg.stats()
    assert og.num_steps() == len(st)
    for s in range(len(st)):
        assert og.step_info(s)["kind"] == st[s]["kind"], s
        for x, y in zip(og.step_output(s), gg.step_output(s)):
            assert np.array_equal(x, y), (w.name, s)
    assert np.array_equal(om, gm) and np.array_equal(ot, gt)
    for i in np.linspace(0, len(om) - 1, strategies).astype(int):
        assert np.array_equal(og.strategy(int(i)), gg.strategy(int(i)))
    lg = ft.load(w)
    lg.eliminate()
    lm, lt = lg.frontier()
    assert np.array_equal(lm, gm) and np.array_equal(lt, gt)
    return st


def test_ft_elimination(ft):
    for seed in range(20):
        compare_elim(ft, G.random_sp(700 + seed, n_ops=3 + seed % 10, kmax=6, cost_hi=1 << 12))
    for var in ("chain", "parallel", "diamond"):
        compare_elim(ft, G.c1(3, var))
    compare_elim(ft, G.c2())
    compare_elim(ft, G.c3())
    st = compare_elim(ft, G.c4(layers=2))
    assert st[-1]["kind"] == "pair" and st[-1]["nblk"] == 36 * 36
    with pytest.raises(ft.FTError):
        g = ft.load(G.c1(0, "chain"))
        g.eliminate()
        g.frontier(algo="elim")
        g.frontier()  # the graph's frontier was computed by FT-Elimination


def test_branch_elimination(ft):
    """Branch elimination (Eq. 6) in FT_AUTO: graphs with attached input and
    output ops; every step bit-identical to the oracle, for FT-LDP and
    FT-Elimination."""
    kinds = set()
    for seed in range(30):
        w = G.random_leafy(seed, n_ops=2 + seed % 6, kmax=6, leaves=1 + seed % 4, cost_hi=1 << 12)
        _, st = compare(ft, w, strategies=8)
        kinds |= {s["kind"] for s in st}
        compare_elim(ft, w, strategies=4)
    assert "branch" in kinds
    compare(ft, G.random_graph(3, [(0, 2), (1, 2)], 40, 5, cost_hi=1 << 20), strategies=8)


def test_mini_time_query(ft):
    """ft_query_mini_time (SS4.1) returns the oracle's index at every limit."""
    for w in (G.c2(), G.c3(), G.random_sp(77, n_ops=12, kmax=6, cost_hi=1 << 16)):
        og = oracle.load(w, 8)
        og.eliminate()
        om, _ = og.frontier()
        g = ft.load(w)
        g.eliminate()
        gm, _ = g.frontier()
        lims = [int(om[0]) - 1] + om.tolist() + (om + 1).tolist() + [1 << 62]
        for lim in lims:
            assert g.mini_time(lim) == og.mini_time(lim), lim
        i = g.mini_time(int(om[len(om) // 2]))
        assert np.array_equal(g.strategy(i), og.strategy(i))


def test_heuristic_elimination(ft):
    """FT_AUTO_HEUR (Eq. 7 heuristic elimination, lossy): the GPU applies the
    oracle's rule and matches it step by step; includes BERT with a K=36 mask."""
    import paper_2004_10856_b200 as ftm
    n = 0
    for seed in range(24):
        w = G.random_masked(seed, n_ops=3 + seed % 5, kmax=4, mask_k=2 + seed % 3, fanout=2 + seed % 2)
        og = oracle.load(w, 4)
        og.eliminate(oracle.AUTO_HEUR)
        try:
            om, ot = og.frontier()
        except oracle.OracleError:
            continue
        g = ft.load(w, keep_all=True)
        g.eliminate(ftm.AUTO_HEUR)
        gm, gt = g.frontier()
        assert np.array_equal(om, gm) and np.array_equal(ot, gt)
        assert og.num_steps() == len(g.stats())
        for s in range(og.num_steps()):
            for x, y in zip(og.step_output(s), g.step_output(s)):
                assert np.array_equal(x, y), (seed, s)
        for i in range(len(om)):
            assert np.array_equal(og.strategy(i), g.strategy(i))
        n += 1
    assert n > 10
    w = G.c4(layers=2, mask_k1=False)
    og = oracle.load(w, 8)
    og.eliminate(oracle.AUTO_HEUR)
    om, ot = og.frontier()
    g = ft.load(w)
    g.eliminate(ftm.AUTO_HEUR)
    gm, gt = g.frontier()
    assert np.array_equal(om, gm) and np.array_equal(ot, gt)


@pytest.mark.parametrize("world", [2, 3])
def test_partition_invariance_new_kinds(ft, world):
    """Sharded execution (loopback virtual ranks) of branch elimination,
    heuristic elimination and FT-Elimination's pair reduce is bit-identical
    to world = 1."""
    import paper_2004_10856_b200 as ftm
    cases = [(G.random_leafy(5, n_ops=7, kmax=6, leaves=3, cost_hi=1 << 12), ftm.AUTO, "ldp"),
             (G.random_leafy(9, n_ops=6, kmax=6, leaves=2, cost_hi=1 << 12), ftm.AUTO, "elim"),
             (G.c4(layers=2, mask_k1=False), ftm.AUTO_HEUR, "ldp"),
             (G.c3(), ftm.AUTO, "elim")]
    for w, kind, algo in cases:
        a = ft.load(w, keep_all=True)
        a.eliminate(kind)
        am, at = a.frontier(algo=algo)
        b = ft.load(w, keep_all=True, world=world, loopback=True)
        b.eliminate(kind)
        bm, bt = b.frontier(algo=algo)
        assert np.array_equal(am, bm) and np.array_equal(at, bt), w.name
        for s in range(len(a.stats())):
            for x, y in zip(a.step_output(s), b.step_output(s)):
                assert np.array_equal(x, y), (w.name, s)


# ---- R10 range: frontier m up to 2^60 (packed single-key sorts must stay exact)

def test_big_chain_wide_costs(ft):
    """16,384-op chain, K = 2, every op and edge cost (memory included) just
    below 2^40: frontier m ~ 2^55, beyond what an unshifted (m << 10 | e) key
    holds.  Every step bit-exact against the oracle."""
    w = G.big_chain(n_ops=16384)
    gg, st = compare(ft, w, strategies=48)
    assert gg.frontier()[0][0] > 1 << 54


def test_bert_2layers_scaled_to_2_40(ft):
    """BERT-2L with every cost scaled just below 2^40 (R10's input bound)."""
    compare(ft, G.scaled(G.c4(layers=2)), strategies=32)


@pytest.mark.parametrize("bits", ["0", "12"])
def test_full_key_sort_fallback(ft, monkeypatch, bits):
    """FT_KEY_SPAN_BITS forces the full (m, t, id) sorts that take over when a
    sample's m span does not fit the packed key: every step still exact, and
    the shared-order node rows go to the full-key CTA kernel."""
    monkeypatch.setenv("FT_KEY_SPAN_BITS", bits)
    for w in (G.c3(), G.c4(layers=2), G.c5(n_ops=300, K=32, B=8, Lmin=3, Lmax=8),
              G.scaled(G.random_sp(1003, n_ops=14, kmax=12, cost_hi=1 << 20))):
        gg, st = compare(ft, w, strategies=16)
        if w.name.startswith("C5"):
            assert sum(s["path"]["shared_cta_rows"] for s in st) > 0  # rows handed to k_node_shared


# ---- branch elimination with composite configurations (Eq. 6, R21)

def test_bridge_and_random_dags_composite(ft):
    """Non-series-parallel DAGs linearised by composite branch elimination:
    every step (compose, remap, ...) bit-exact against the oracle, composite
    configurations split back in every strategy."""
    n = 0
    for K in (2, 3, [2, 3, 4, 2], [3, 4, 1, 2], 40):
        w = G.random_graph(4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], K, 3, cost_hi=1 << 20, edge_mem=True)
        gg, st = compare(ft, w)
        n += any(s["kind"] == "compose" for s in st)
    skipped = 0
    for seed in range(120):
        w = G.random_dag(seed, n_ops=3 + seed % 9, kmax=4 + seed % 5, p_edge=0.35,
                         cost_hi=1 << (4 + seed % 20), edge_mem=(seed % 4 == 0))
        og = oracle.load(w, 4)
        og.eliminate()
        try:
            og.frontier()
        except oracle.OracleError as e:  # composite spaces would exceed 4096: not linearisable
            assert e.code == oracle.EPRECOND
            g = ft.load(w)
            g.eliminate()
            with pytest.raises(ft.FTError) as fe:
                g.frontier()
            assert fe.value.code == ft.EPRECOND
            skipped += 1
            continue
        gg, st = compare(ft, w, strategies=8)
        n += any(s["kind"] == "compose" for s in st)
    assert n >= 50 and skipped < 40


def test_composite_loopback_and_elimination(ft):
    """Composite graphs sharded over virtual ranks, and FT-Elimination on them."""
    for seed in (5, 17, 29):
        w = G.random_dag(seed, n_ops=10, kmax=6, p_edge=0.3, cost_hi=1 << 16)
        a = ft.load(w, keep_all=True)
        a.eliminate()
        am, at = a.frontier()
        b = ft.load(w, keep_all=True, world=3, loopback=True)
        b.eliminate()
        bm, bt = b.frontier()
        assert np.array_equal(am, bm) and np.array_equal(at, bt)
        c = ft.load(w)
        c.eliminate()
        cm, ct = c.frontier(algo="elim")
        og = oracle.load(w, 4)
        og.eliminate()
        om, ot = og.frontier(algo="elim")
        assert np.array_equal(cm, om) and np.array_equal(ct, ot) and np.array_equal(cm, am)


@pytest.mark.parametrize("alpha", [(1, 2), (1, 5), (0, 1)])
def test_weighted_heuristic(ft, alpha):
    """FT_HEUR_WEIGHTED (R22): the GPU library picks the oracle's
    configuration and matches it step by step."""
    n = 0
    for seed in range(16):
        w = G.random_masked(seed, n_ops=3 + seed % 5, kmax=4, mask_k=2 + seed % 3, fanout=2 + seed % 2,
                            cost_hi=1 << 12)
        og = oracle.load(w, 4)
        og.set_heuristic("weighted", alpha)
        og.eliminate(oracle.AUTO_HEUR)
        try:
            om, ot = og.frontier()
        except oracle.OracleError:
            continue
        g = ft.load(w, keep_all=True)
        g.set_heuristic("weighted", alpha)
        g.eliminate(ft.AUTO_HEUR)
        gm, gt = g.frontier()
        assert np.array_equal(om, gm) and np.array_equal(ot, gt)
        for s in range(og.num_steps()):
            for x, y in zip(og.step_output(s), g.step_output(s)):
                assert np.array_equal(x, y), (seed, s)
        for i in range(len(om)):
            assert np.array_equal(og.strategy(i), g.strategy(i))
        n += 1
    assert n > 6


def test_composite_max_k_and_heur_fallback(ft):
    """Composite configurations at the library's bound (K_h * K_i = 4096:
    4,096-configuration operator, wide segments downstream), and FT_AUTO_HEUR
    falling back to a composite when no source can be fixed (R21)."""
    bridge = [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)]
    w = G.random_graph(4, bridge, [3, 64, 64, 5], 7, cost_hi=1 << 30)
    gg, st = compare(ft, w, strategies=16)
    assert any(s["kind"] == "compose" and s["nseg"] == 4096 for s in st)
    w = G.random_graph(5, bridge + [(3, 4)], [2, 3, 4, 3, 2], 11, cost_hi=1 << 16)
    og = oracle.load(w, 4)
    og.eliminate(oracle.AUTO_HEUR)
    om, ot = og.frontier()
    g = ft.load(w, keep_all=True)
    g.eliminate(ft.AUTO_HEUR)
    gm, gt = g.frontier()
    assert np.array_equal(om, gm) and np.array_equal(ot, gt)
    assert any(s["kind"] == "compose" for s in g.stats())
    for i in range(len(om)):
        assert np.array_equal(og.strategy(i), g.strategy(i))
