"""Pins for branch elimination (Eq. 6) in the
oracle's FT_AUTO policy: an unmarked op whose only edge connects it to one
neighbour o_h is merged into o_h, reducing over its configurations at once
(reading R14).  Exact, so brute force (Def. 1)
must agree on tiny graphs and every unrolled strategy must re-cost (Eq. 3)."""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
from synth import graphs as G


def _run(w, algo="ldp"):
    g = oracle.load(w, 4)
    g.eliminate()
    m, t = g.frontier(algo=algo)
    kinds = [g.step_info(s)["kind"] for s in range(g.num_steps())]
    return g, m, t, kinds


@pytest.mark.parametrize("seed", range(60))
def test_branch_brute_force(seed):
    w = G.random_leafy(seed, n_ops=2 + seed % 4, kmax=3, leaves=1 + seed % 3, edge_mem=(seed % 5 == 0))
    if int(np.prod([int(k) for k in w.n_cfgs], dtype=np.int64)) > 200_000:
        pytest.skip("too many strategies for brute force")
    g, m, t, _ = _run(w)
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []
    for i in range(len(m)):
        assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))


def test_branch_is_used():
    """Two K>1 inputs of one op: only branch elimination linearises it."""
    w = G.random_graph(3, [(0, 2), (1, 2)], 3, 5)
    g, m, t, kinds = _run(w)
    assert "branch" in kinds
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []


@pytest.mark.parametrize("seed", range(10))
def test_branch_with_elimination_baseline(seed):
    """FT-Elimination after branch eliminations equals FT-LDP (both exact)."""
    w = G.random_leafy(300 + seed, n_ops=6, kmax=5, leaves=3, cost_hi=1 << 12)
    _, m, t, _ = _run(w)
    _, m2, t2, _ = _run(w, algo="elim")
    assert np.array_equal(m, m2) and np.array_equal(t, t2)


def test_branch_sink_and_source_orientation():
    """A leaf on each side of one op: source leaf (edge i -> h) and sink leaf
    (edge h -> i) index the edge table differently (Eq. 2 row-major)."""
    w = G.random_graph(4, [(0, 1), (2, 1), (1, 3)], [2, 3, 4, 2], 11, cost_hi=50)
    g, m, t, kinds = _run(w)
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []
    for i in range(len(m)):
        assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))
