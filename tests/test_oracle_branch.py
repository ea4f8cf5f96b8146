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


# ---- composite configurations (Eq. 6 with o_i keeping other edges, R21)

BRIDGE = [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)]


@pytest.mark.parametrize("K", [2, 3, [2, 3, 4, 2], [3, 4, 1, 2]])
def test_bridge_dag_composite(K):
    """The bridge DAG is not series-parallel: no node, edge, fold or leaf
    branch elimination applies.  Merging o_1 into o_2 (composite configs
    (s_2, s_1)) makes it a chain; the frontier equals brute force and every
    unrolled strategy -- composites split back -- re-costs exactly."""
    w = G.random_graph(4, BRIDGE, K, 3, cost_hi=40, edge_mem=True)
    g, m, t, kinds = _run(w)
    assert kinds.count("compose") == 1 and kinds.count("remap") == 4
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []
    for i in range(len(m)):
        assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))


@pytest.mark.parametrize("seed", range(200))
def test_random_dag_composite_brute_force(seed):
    """Random (mostly non-series-parallel) DAGs: FT_AUTO with composite
    branch elimination is exact -- Def. 1 against the enumeration, re-cost of
    every strategy -- and FT-Elimination agrees with FT-LDP."""
    w = G.random_dag(seed, n_ops=3 + seed % 6, kmax=3, p_edge=0.35, edge_mem=(seed % 4 == 0))
    if int(np.prod([int(k) for k in w.n_cfgs], dtype=np.int64)) > 100_000:
        pytest.skip("too many strategies for brute force")
    g, m, t, kinds = _run(w)
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []
    for i in range(len(m)):
        assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))
    _, m2, t2, _ = _run(w, algo="elim")
    assert np.array_equal(m, m2) and np.array_equal(t, t2)


def test_composite_used_on_most_random_dags():
    used = 0
    for seed in range(60):
        w = G.random_dag(seed, n_ops=6, kmax=3, p_edge=0.35)
        _, _, _, kinds = _run(w)
        used += "compose" in kinds
    assert used >= 20


def test_composite_cap_and_cycle_guard():
    """K_h * K_i > 4096 is refused (the graph stays non-linear: FT_EPRECOND);
    an input o_i with another path to o_h is never merged into it (it would
    close a cycle) -- here o_1 -> o_2 -> o_3 and o_1 -> o_3: o_2 is
    node-eliminated first instead (series), so no composite is needed."""
    w = G.random_graph(4, BRIDGE, 65, 0)
    g = oracle.load(w)
    g.eliminate()
    with pytest.raises(oracle.OracleError):
        g.frontier()
    w = G.random_graph(4, [(0, 1), (1, 2), (2, 3), (1, 3), (0, 3)], 3, 1)
    g, m, t, kinds = _run(w)
    ma, ta, _ = bf.enumerate_costs(w)
    assert bf.check_frontier(m, t, ma, ta) == []
