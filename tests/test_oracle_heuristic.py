"""Pins for heuristic elimination (Eq. 7),
opt-in via OFT_AUTO_HEUR.  It is lossy in general, so the exact pin is on
the RESTRICTED problem: with the mask op fixed to the configuration the rule
picks (least memory, ties by time then index -- computed here from the cost
tables), the frontier must equal brute force over that restricted strategy
space; and every point must be achievable in the full problem (quality is
reported as the share of the exact frontier it reproduces)."""
import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf
from synth import graphs as G


def _restricted(w, op, k):
    """Workload with op's configuration fixed to k (Eq. 1 / Eq. 2 slices)."""
    K = w.n_cfgs.copy()
    op_m = list(w.op_m)
    op_t = list(w.op_t)
    op_m[op] = w.op_m[op][k:k + 1].copy()
    op_t[op] = w.op_t[op][k:k + 1].copy()
    edge_t = list(w.edge_t)
    edge_m = None if w.edge_m is None else list(w.edge_m)
    for e in range(w.n_edges):
        s, d = int(w.src[e]), int(w.dst[e])
        if s == op:
            sl = slice(k * int(K[d]), (k + 1) * int(K[d]))
        elif d == op:
            sl = slice(k, None, int(K[op]))
        else:
            continue
        edge_t[e] = w.edge_t[e][sl].copy()
        if edge_m is not None:
            edge_m[e] = w.edge_m[e][sl].copy()
    K[op] = 1
    return G.Workload(w.name + "-fixed", K, w.src, w.dst, op_m, op_t, edge_t, edge_m).check()


def _ok(w):
    g = oracle.load(w, 2)
    g.eliminate(oracle.AUTO_HEUR)
    try:
        m, t = g.frontier()
    except oracle.OracleError as e:
        assert e.code == oracle.EPRECOND  # heuristics only remove sources
        return None
    return g, m, t


@pytest.mark.parametrize("seed", range(40))
def test_heuristic_restricted_brute_force(seed):
    w = G.random_masked(seed, n_ops=3 + seed % 4, kmax=3, mask_k=2 + seed % 2, fanout=2 + seed % 2)
    r = _ok(w)
    if r is None:
        pytest.skip("not linearisable by source heuristics")
    g, m, t = r
    mask = w.n_ops - 1
    # FT_AUTO_HEUR tries heuristic elimination before composite branch
    # elimination (R17, R21): either the mask was fixed (then the result is
    # exact on the restricted space) or no heuristic ran (then it is exact)
    ma, ta, _ = bf.enumerate_costs(w)
    if bf.check_frontier(m, t, ma, ta) == []:
        return
    om, ot = w.op_m[mask], w.op_t[mask]
    ks = min(range(len(om)), key=lambda k: (int(om[k]), int(ot[k]), k))
    wr = _restricted(w, mask, ks)
    ma, ta, _ = bf.enumerate_costs(wr)
    assert bf.check_frontier(m, t, ma, ta) == []       # exact on the restricted space
    for i in range(len(m)):
        s = g.strategy(i)
        assert s[mask] == ks
        assert bf.total_cost(w, s) == (int(m[i]), int(t[i]))  # achievable in the full problem


def test_heuristic_quality_report():
    """Share of the exact frontier the heuristic reproduces (lossy by design)."""
    got = tot = 0
    for seed in range(20):
        w = G.random_masked(seed, n_ops=4, kmax=3, mask_k=3, fanout=3)
        r = _ok(w)
        if r is None:
            continue
        _, m, t = r
        ex = bf.brute_force(w)
        pts = set(zip(m.tolist(), t.tolist()))
        got += sum((a, b) in pts for a, b in ex)
        tot += len(ex)
    assert tot > 0 and 0 < got <= tot


def test_heuristic_off_by_default():
    """FT_AUTO never applies it: the K>1-mask BERT graph stays non-linear."""
    w = G.c4(layers=2, mask_k1=False)  # (one layer: the mask is a leaf -> exact branch elimination)
    g = oracle.load(w, 8)
    g.eliminate(oracle.AUTO)
    with pytest.raises(oracle.OracleError) as e:
        g.frontier()
    assert e.value.code == oracle.EPRECOND
    g = oracle.load(w, 8)
    g.eliminate(oracle.AUTO_HEUR)
    m, t = g.frontier()
    assert len(m) > 0


def _weighted_choice(w, op, alpha):
    """R22's rule written out from the cost tables (IEEE double, each
    operation rounded once -- Python floats): least alpha*m/M + (1-alpha)*t/T."""
    m = [int(x) for x in w.op_m[op]]
    t = [int(x) for x in w.op_t[op]]
    M, T = max(1, max(m)), max(1, max(t))
    al = alpha[0] / alpha[1]
    key = lambda k: (al * (m[k] / M) + (1.0 - al) * (t[k] / T), m[k], t[k], k)
    return min(range(len(m)), key=key)


@pytest.mark.parametrize("alpha", [(1, 2), (1, 4), (3, 4), (0, 1), (1, 1)])
@pytest.mark.parametrize("seed", range(24))
def test_weighted_heuristic_restricted_brute_force(seed, alpha):
    """P:622 "a weighted combination of different objectives" (reading R22):
    exact on the restricted problem with the mask fixed to the rule's pick."""
    w = G.random_masked(seed, n_ops=3 + seed % 4, kmax=3, mask_k=2 + seed % 3, fanout=2 + seed % 2,
                        cost_hi=40)
    g = oracle.load(w, 2)
    g.set_heuristic("weighted", alpha)
    g.eliminate(oracle.AUTO_HEUR)
    try:
        m, t = g.frontier()
    except oracle.OracleError:
        pytest.skip("not linearisable")
    ma, ta, _ = bf.enumerate_costs(w)
    if bf.check_frontier(m, t, ma, ta) == []:
        return  # no heuristic step was needed
    mask = w.n_ops - 1
    ks = _weighted_choice(w, mask, alpha)
    ma, ta, _ = bf.enumerate_costs(_restricted(w, mask, ks))
    assert bf.check_frontier(m, t, ma, ta) == []
    for i in range(len(m)):
        s = g.strategy(i)
        assert s[mask] == ks and bf.total_cost(w, s) == (int(m[i]), int(t[i]))


def test_weighted_alpha_one_is_least_memory():
    """alpha = 1 scores m/M: the same pick as the least-memory rule (ties by t)."""
    for seed in range(30):
        w = G.random_masked(seed, n_ops=5, kmax=3, mask_k=4, fanout=3, cost_hi=40)
        res = []
        for pol in ("min_memory", "weighted"):
            g = oracle.load(w, 2)
            g.set_heuristic(pol, (1, 1))
            g.eliminate(oracle.AUTO_HEUR)
            try:
                res.append(g.frontier())
            except oracle.OracleError:
                res.append(None)
        if res[0] is not None:
            assert all(np.array_equal(a, b) for a, b in zip(res[0], res[1]))


def test_set_heuristic_errors():
    w = G.random_masked(0)
    g = oracle.load(w)
    for bad in ((2, 1), (-1, 2), (1, 0)):
        with pytest.raises(oracle.OracleError):
            g.set_heuristic("weighted", bad)


def quality(policy, alpha=(1, 2), n=50):
    """S:603 acceptance criterion 3 on n shared-input fixtures: every returned
    tuple is feasible (re-costs exactly) and the output is mutually
    non-dominated; returns the mean fraction of oracle (exact, brute-force)
    frontier points that the heuristic output weakly dominates."""
    fr = []
    for seed in range(n):
        w = G.random_masked(1000 + seed, n_ops=4 + seed % 3, kmax=3, mask_k=3, fanout=3, cost_hi=40)
        g = oracle.load(w, 2)
        g.set_heuristic(policy, alpha)
        g.eliminate(oracle.AUTO_HEUR)
        try:
            m, t = g.frontier()
        except oracle.OracleError:
            continue
        for i in range(len(m)):
            assert bf.total_cost(w, g.strategy(i)) == (int(m[i]), int(t[i]))
        assert (np.diff(m) > 0).all() and (np.diff(t) < 0).all()
        ex = bf.brute_force(w)
        fr.append(sum(bool(((m <= a) & (t <= b)).any()) for a, b in ex) / len(ex))
    return float(np.mean(fr)), len(fr)


def test_heuristic_quality_s603():
    for pol in ("min_memory", "weighted"):
        q, n = quality(pol)
        assert n >= 40 and 0.0 < q <= 1.0, (pol, q, n)
