"""Pins for the oracle's FT driver: brute force on tiny graphs,
scalar min-plus DPs on the large configs, frontier invariants."""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
from oracle import scalar_dp as sdp
from synth import graphs as G


def _workload_from_case(case):
    K = np.asarray(case["K"], np.int32)
    edges = case["edges"]
    return G.Workload(case["id"], K, np.asarray([e[0] for e in edges], np.int32),
                      np.asarray([e[1] for e in edges], np.int32),
                      [np.asarray(x, np.int64) for x in case["op_m"]],
                      [np.asarray(x, np.int64) for x in case["op_t"]],
                      [np.asarray(x, np.int64) for x in case["edge_t"]]).check()


def test_total_cost_golden(golden):
    for case in golden["total_cost"]:
        w = _workload_from_case(case)
        assert list(bf.total_cost(w, case["strategy"])) == case["expected"]


def test_graph_golden(golden):
    for case in golden["graphs"]:
        w = _workload_from_case(case)
        g, m, t = oracle.run_ft(w)
        assert [[int(a), int(b)] for a, b in zip(m, t)] == case["expected_frontier"], case["id"]
        if "expected_strategy" in case:
            assert [g.strategy(i).tolist() for i in range(len(m))] == case["expected_strategy"]


def _check_vs_bruteforce(w):
    g, m, t = oracle.run_ft(w)
    assert list(zip(m.tolist(), t.tolist())) == bf.brute_force(w)
    for i in range(len(m)):
        assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))


@pytest.mark.parametrize("variant", ["chain", "parallel", "diamond"])
def test_c1_vs_bruteforce(variant):
    """C1 (BASELINE configs[0]), 1,000 seeds per variant: (m,t) set equality
    with the Def. 1 brute-force frontier and Eq. 3 re-cost of every strategy."""
    for seed in range(1000):
        _check_vs_bruteforce(G.c1(seed, variant))


@pytest.mark.parametrize("seed", range(300))
def test_random_sp_vs_bruteforce(seed):
    w = G.random_sp(seed, n_ops=2 + seed % 8, kmax=3, edge_mem=(seed % 5 == 0))
    if int(np.prod(w.n_cfgs.astype(np.int64))) > 200_000:
        pytest.skip("too many strategies")
    _check_vs_bruteforce(w)


def test_enumeration_def1_check():
    """Def. 1 checked against the whole enumeration without sorting."""
    for seed in range(30):
        w = G.random_sp(100 + seed, n_ops=7, kmax=3)
        if int(np.prod(w.n_cfgs.astype(np.int64))) > 200_000:
            continue
        _, m, t = oracle.run_ft(w)
        ma, ta, _ = bf.enumerate_costs(w)
        assert bf.check_frontier(m, t, ma, ta) == []


def _large_pins(w, m, t):
    assert (np.diff(m) > 0).all() and (np.diff(t) < 0).all()
    assert (int(m[0]), int(t[0])) == sdp.min_memory_endpoint(w)
    assert int(m[0]) == sdp.min_memory_closed_form(w)
    assert (int(m[-1]), int(t[-1])) == sdp.min_time_endpoint(w)
    for a, b in [(1, 4), (1, 1), (3, 1), (0, 1), (1, 0)]:
        assert int(np.min(b * t + a * m)) == sdp.weighted_optimum(w, a, b), (a, b)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_large_configs_scalar_pins(name):
    w = G.get(name)
    g, m, t = oracle.run_ft(w, threads=4)
    _large_pins(w, m, t)
    # sampled strategies re-cost exactly
    for i in np.linspace(0, len(m) - 1, 12).astype(int):
        assert bf.total_cost(w, g.strategy(int(i))) == (int(m[i]), int(t[i]))
    # random strategies are dominated by some frontier tuple (north-star invariant)
    rng = np.random.default_rng(3)
    for _ in range(300):
        S = [int(rng.integers(0, k)) for k in w.n_cfgs]
        sm, st = bf.total_cost(w, S)
        assert ((m <= sm) & (t <= st)).any()


def test_bert_small_mask_fold_pins():
    """C4 structure at 2 layers (mask = K=1 source folded, R13)."""
    w = G.c4(layers=2)
    g, m, t = oracle.run_ft(w, threads=4)
    _large_pins(w, m, t)
    steps = [g.step_info(s)["kind"] for s in range(g.num_steps())]
    assert steps.count("fold") == 2
    for i in np.linspace(0, len(m) - 1, 8).astype(int):
        assert bf.total_cost(w, g.strategy(int(i))) == (int(m[i]), int(t[i]))


def test_c5_small_pins():
    """C5 generator at reduced size (120 ops, K=8)."""
    w = G.c5(n_ops=120, K=8, B=6, Lmin=2, Lmax=5)
    g, m, t = oracle.run_ft(w, threads=4)
    _large_pins(w, m, t)
    for i in np.linspace(0, len(m) - 1, 8).astype(int):
        assert bf.total_cost(w, g.strategy(int(i))) == (int(m[i]), int(t[i]))


def test_thread_count_invariance():
    w = G.c3()
    g1 = oracle.load(w, threads=1)
    g1.eliminate()
    g4 = oracle.load(w, threads=8)
    g4.eliminate()
    assert g1.num_steps() == g4.num_steps()
    for s in range(0, g1.num_steps(), 7):
        a = g1.step_output(s)
        b = g4.step_output(s)
        for x, y in zip(a, b):
            assert (x == y).all()


# ---- R10 range: costs just below 2^40, frontier m far beyond 2^40

@pytest.mark.parametrize("seed", range(40))
def test_scaled_costs_vs_bruteforce(seed):
    """Tiny graphs with every cost scaled just below 2^40 (edge memory too):
    brute force in Python ints (Eq. 3, Def. 1)."""
    w = G.scaled(G.random_sp(seed, n_ops=2 + seed % 7, kmax=3, edge_mem=(seed % 3 == 0)))
    if int(np.prod(w.n_cfgs.astype(np.int64))) > 100_000:
        pytest.skip("too many strategies")
    _check_vs_bruteforce(w)


def test_big_chain_scalar_pins():
    """Wide-cost chain (1,024 ops; m ~ 2^50): endpoints and supported points
    by the scalar DPs in exact integers."""
    w = G.big_chain(n_ops=1024)
    g, m, t = oracle.run_ft(w, threads=4)
    assert (np.diff(m) > 0).all() and (np.diff(t) < 0).all() and int(m[0]) > 1 << 49
    assert (int(m[0]), int(t[0])) == sdp.min_memory_endpoint(w)
    assert (int(m[-1]), int(t[-1])) == sdp.min_time_endpoint(w)
    M, T = [int(x) for x in m], [int(x) for x in t]
    for a, b in [(1, 4), (1, 1), (3, 1), (1 << 30, 1)]:
        assert min(b * y + a * x for x, y in zip(M, T)) == sdp.weighted_optimum(w, a, b), (a, b)
    for i in np.linspace(0, len(m) - 1, 6).astype(int):
        assert bf.total_cost(w, g.strategy(int(i))) == (M[i], T[i])
