"""Pins for the mini-time frontier query (SS4.1):
the answer must be the minimum time over ALL strategies with m <= limit
(brute force, Eq. 3), or infeasible below the minimum memory."""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
from synth import graphs as G


@pytest.mark.parametrize("seed", range(30))
def test_mini_time_brute_force(seed):
    w = G.random_sp(1200 + seed, n_ops=2 + seed % 5, kmax=3, cost_hi=50)
    g = oracle.load(w, 2)
    g.eliminate()
    m, t = g.frontier()
    ma, ta, _ = bf.enumerate_costs(w)
    limits = sorted(set([int(ma.min()) - 1, int(ma.max()) + 1] + m.tolist() +
                        (m[:-1] + 1).tolist() if len(m) > 1 else [int(ma.min()) - 1, int(ma.max())]))
    for lim in limits:
        i = g.mini_time(lim)
        feas = ma <= lim
        if not feas.any():
            assert i == -1
            continue
        assert i >= 0 and int(m[i]) <= lim
        assert int(t[i]) == int(ta[feas].min())          # fastest strategy that fits
        assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))


def test_mini_time_examples():
    """SPEC S:497-500 shapes: unconstrained -> global min time; below the
    smallest memory -> infeasible."""
    w = G.c2()
    g = oracle.load(w, 8)
    g.eliminate()
    m, t = g.frontier()
    assert g.mini_time(1 << 62) == len(m) - 1
    assert g.mini_time(int(m[0]) - 1) == -1
    assert g.mini_time(int(m[0])) == 0
