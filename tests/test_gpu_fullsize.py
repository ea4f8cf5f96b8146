"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration.

* C4 (BERT-large, 5.8e9 product tuples): the oracle runs the whole search;
  every step output (seg_off, m, t, bp), the final frontier and sampled
  strategies must be bit-identical.
* C5 (2,000-op SP DAG, 2.7e10 tuples): the oracle recomputes sampled output
  segments one by one (``oft_segment_reduce``) from the factor frontiers that
  the GPU step consumed (``ft_step_inputs`` + earlier step outputs / original
  costs, block mapping written from Eq. 4 / Eq. 5 / Eq. 7 / Alg. 3); the final
  frontier is pinned by the scalar DPs (endpoints, supported points) and every
  sampled strategy re-costs exactly (Eq. 3).
"""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
from oracle import scalar_dp as sdp
from synth import graphs as G

pytestmark = pytest.mark.gpu

NODE, EDGE, FOLD, LDP, FINAL = 1, 2, 3, 4, 5


@pytest.fixture(scope="module")
def ft():
    import paper_2004_10856_b200 as ft
    return ft


def _factor(g, w, src, seg, cache):
    """(m[], t[]) of segment `seg` of a factor set described by ft_step_inputs."""
    kind, ident = int(src[0]), int(src[1])
    if kind == 0:
        return np.zeros(1, np.int64), np.zeros(1, np.int64)
    if kind == 1:
        return w.op_m[ident][seg:seg + 1], w.op_t[ident][seg:seg + 1]
    if kind == 2:
        em = np.zeros(1, np.int64) if w.edge_m is None else w.edge_m[ident][seg:seg + 1]
        return em, w.edge_t[ident][seg:seg + 1]
    if ident not in cache:
        so, m, t, _ = g.step_output(ident)
        cache[ident] = (so, m, t)
    so, m, t = cache[ident]
    return m[so[seg]:so[seg + 1]], t[so[seg]:so[seg + 1]]


def _blocks(par, sigma):
    """Factor segments (x, y, z) of every block of output segment sigma."""
    kind, KA, KB, KC, nseg, nblk = (int(v) for v in par)
    out = []
    for k in range(nblk):
        if kind == NODE:      # Eq. 4: sigma = w*K_j + p
            wv, p = divmod(sigma, KC)
            out.append((wv * KB + k, k, k * KC + p))
        elif kind == LDP:     # Alg. 3 line 6: sigma = p
            out.append((k * KB + sigma, k, sigma))
        elif kind == FINAL:   # Alg. 3 line 9
            out.append((k, 0, 0))
        else:                 # Eq. 5 / Eq. 7
            out.append((sigma, sigma, 0))
    return out


def check_sampled_segments(g, w, steps, per_step=3, seed=0):
    rng = np.random.default_rng(seed)
    cache = {}
    checked = 0
    for s in steps:
        src, par = g.step_inputs(s)
        so, m, t, bp = g.step_output(s)
        nseg = int(par[4])
        segs = sorted(set([0, nseg - 1] + rng.integers(0, nseg, per_step).tolist()))
        for sg in segs:
            blocks = []
            for (sx, sy, sz) in _blocks(par, sg):
                blocks.append((_factor(g, w, src[0], sx, cache), _factor(g, w, src[1], sy, cache),
                               _factor(g, w, src[2], sz, cache)))
            om, ot, oid = oracle.segment_reduce(blocks)
            gm, gt, gb = m[so[sg]:so[sg + 1]], t[so[sg]:so[sg + 1]], bp[so[sg]:so[sg + 1]]
            assert np.array_equal(om, gm) and np.array_equal(ot, gt) and np.array_equal(oid, gb), \
                (s, sg)
            checked += 1
        cache.pop(s, None)
    return checked


def final_pins(g, w, m, t, n_strat=24):
    assert (np.diff(m) > 0).all() and (np.diff(t) < 0).all()
    assert (int(m[0]), int(t[0])) == sdp.min_memory_endpoint(w)
    assert (int(m[-1]), int(t[-1])) == sdp.min_time_endpoint(w)
    for a, b in [(1, 4), (1, 1), (3, 1)]:
        assert int(np.min(b * t + a * m)) == sdp.weighted_optimum(w, a, b), (a, b)
    for i in np.linspace(0, len(m) - 1, n_strat).astype(int):
        assert bf.total_cost(w, g.strategy(int(i))) == (int(m[i]), int(t[i]))


def test_c4_full_every_step(ft):
    w = G.c4()
    og = oracle.load(w, threads=0 or 64)
    og.eliminate()
    om, ot = og.frontier()
    g = ft.load(w, keep_all=True)
    g.eliminate()
    gm, gt = g.frontier()
    st = g.stats()
    assert og.num_steps() == len(st)
    for s in range(len(st)):
        for x, y in zip(og.step_output(s), g.step_output(s)):
            assert np.array_equal(x, y), s
    assert np.array_equal(om, gm) and np.array_equal(ot, gt)
    for i in np.linspace(0, len(om) - 1, 48).astype(int):
        assert np.array_equal(og.strategy(int(i)), g.strategy(int(i)))
    final_pins(g, w, gm, gt, n_strat=8)


def test_c5_full_sampled_segments(ft):
    w = G.c5()
    g = ft.load(w, keep_all=True)
    g.eliminate()
    m, t = g.frontier()
    st = g.stats()
    n = len(st)
    big = sorted(range(n), key=lambda s: -st[s]["tuples"])[:4]
    kinds = {}
    for s in range(n):
        kinds.setdefault(st[s]["kind"], []).append(s)
    sample = set(big) | set(range(0, n, max(1, n // 40)))
    for k, ids in kinds.items():
        sample |= set(ids[:2] + ids[-2:])
    checked = check_sampled_segments(g, w, sorted(sample))
    assert checked > 100
    final_pins(g, w, m, t)


def test_c5_full_every_step(ft):
    """C5 (configs[4], the bench workload) end to end against the oracle run
    over the whole search on every host core: every step's (seg_off, m, t,
    bp), the final frontier and 48 strategies bit-identical (node /
    edge elimination and LDP preserve the exact frontier)."""
    import os
    w = G.c5()
    og = oracle.load(w, threads=len(os.sched_getaffinity(0)))
    og.eliminate()
    om, ot = og.frontier()
    g = ft.load(w, keep_all=True)
    g.eliminate()
    gm, gt = g.frontier()
    st = g.stats()
    assert og.num_steps() == len(st)
    for s in range(len(st)):
        info = og.step_info(s)
        assert info["tuples"] == st[s]["tuples"], s
        for name, x, y in zip(("seg_off", "m", "t", "bp"), og.step_output(s), g.step_output(s)):
            assert np.array_equal(x, y), (s, info["kind"], name)
    assert np.array_equal(om, gm) and np.array_equal(ot, gt)
    for i in np.linspace(0, len(om) - 1, 48).astype(int):
        assert np.array_equal(og.strategy(int(i)), g.strategy(int(i)))


@pytest.mark.parametrize("policy,layers", [("min_memory", 24), ("weighted", 6)])
def test_c4_full_k36_mask_heuristic(ft, policy, layers):
    """BERT-large (C4; all 24 layers for the default rule) with a K = 36
    attention mask: only heuristic elimination linearises it.
    Every step bit-exact against the oracle under both configuration rules
    (R17, R22)."""
    import os
    import paper_2004_10856_b200 as ftm
    w = G.c4(mask_k1=False, layers=layers)
    og = oracle.load(w, threads=len(os.sched_getaffinity(0)))
    og.set_heuristic(policy)
    og.eliminate(oracle.AUTO_HEUR)
    om, ot = og.frontier()
    g = ft.load(w, keep_all=True)
    g.set_heuristic(policy)
    g.eliminate(ftm.AUTO_HEUR)
    gm, gt = g.frontier()
    st = g.stats()
    assert og.num_steps() == len(st)
    assert sum(s["kind"] == "fold" for s in st) == layers  # one heuristic elimination, one fold per consumer
    for s in range(len(st)):
        for x, y in zip(og.step_output(s), g.step_output(s)):
            assert np.array_equal(x, y), s
    assert np.array_equal(om, gm) and np.array_equal(ot, gt)
    for i in np.linspace(0, len(om) - 1, 24).astype(int):
        assert np.array_equal(og.strategy(int(i)), g.strategy(int(i)))
