"""Pins for the oracle's FT-Elimination (Theorem 2), the
SURVEY 8(f) rank-1 "next" row: node-eliminate the linear graph's second op
until two ops remain, then reduce over every configuration pair.

Both FT-LDP and FT-Elimination are exact, so the (m, t)
frontier must equal FT-LDP's and brute force (Def. 1) on tiny graphs;
every unrolled strategy must re-cost exactly (Eq. 3)."""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
from synth import graphs as G

ESTATE = -2


def _elim(w, threads=4):
    g = oracle.load(w, threads)
    g.eliminate()
    n0 = g.num_steps()
    m, t = g.frontier(algo="elim")
    return g, n0, m, t


def _ldp(w, threads=4):
    g = oracle.load(w, threads)
    g.eliminate()
    return g.frontier()


@pytest.mark.parametrize("seed", range(40))
def test_elim_equals_brute_force(seed):
    """Tiny random SP graphs: FT-Elimination == Def. 1 over all strategies."""
    w = G.random_sp(500 + seed, n_ops=2 + seed % 6, kmax=3, edge_mem=(seed % 4 == 0))
    g, _, m, t = _elim(w)
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []
    for i in range(len(m)):
        assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))


@pytest.mark.parametrize("seed", range(12))
def test_elim_equals_ldp(seed):
    """Larger graphs (no brute force): the two exact algorithms agree."""
    w = G.random_sp(900 + seed, n_ops=10 + seed, kmax=6, cost_hi=1 << 16)
    _, _, m, t = _elim(w)
    lm, lt = _ldp(w)
    assert np.array_equal(m, lm) and np.array_equal(t, lt)


@pytest.mark.parametrize("var", ["chain", "parallel", "diamond"])
def test_elim_on_c1(var):
    for seed in range(10):
        w = G.c1(seed, var)
        g, _, m, t = _elim(w)
        lm, lt = _ldp(w)
        assert np.array_equal(m, lm) and np.array_equal(t, lt)
        for i in range(len(m)):
            assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))


def test_elim_step_structure():
    """On a chain of n ops (after FT_AUTO keeps the backbone), FT-Elimination
    runs n-2 node eliminations (second op first) and one pair reduce
    over K_1 * K_n blocks."""
    w = G.c2()  # VGG-16: a 23-op chain
    g, n0, _, _ = _elim(w, threads=8)
    kinds = [g.step_info(s)["kind"] for s in range(n0, g.num_steps())]
    n = w.n_ops
    assert kinds == ["node"] * (n - 2) + ["pair"]
    last = g.step_info(g.num_steps() - 1)
    assert last["nseg"] == 1 and last["nblk"] == int(w.n_cfgs[0]) * int(w.n_cfgs[-1])


def test_elim_single_op():
    w = G.random_sp(3, n_ops=1, kmax=5)
    g, n0, m, t = _elim(w)
    assert [g.step_info(s)["kind"] for s in range(n0, g.num_steps())] == ["final"]
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []


def test_elim_and_ldp_are_exclusive():
    w = G.c1(0, "chain")
    g = oracle.load(w, 1)
    g.eliminate()
    g.frontier(algo="elim")
    with pytest.raises(oracle.OracleError) as ei:
        g.frontier()
    assert ei.value.code == ESTATE
