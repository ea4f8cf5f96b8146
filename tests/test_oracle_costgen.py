"""Pins for the edge-cost generation oracle (
oracle/oracle_costgen.cpp).  Each pin is fixed by the paper's text, a hand
derivation, a closed form or brute force -- not by re-calling the oracle.

* comm_time: P:668-671 ("find the integer i satisfying 2^i <= k < 2^(i+1) and
  use the interpolation of the actual bandwidths at 2^i and 2^(i+1)"), R18.
* split states / re-scheduling: P:860 ("nodes are different tensor splits ...
  the optimal communication operations correspond to the shortest path"), R19.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
from synth import comm


def flat_profile(L=2, P=20, bw=None, lat=0):
    p = comm.profile(0, L=L, P=P)
    p["lat"][:] = 0
    p["lat"][1:L + 1] = lat
    if bw is not None:
        for c in range(1, L + 1):
            p["bw"][c, :] = bw
    return p


def test_comm_time_spec_midpoint():
    # SPEC.md comm_time example: profile {(10, 1e9), (11, 2e9)}, latency 0,
    # 1536 bytes -> 1536 / 1.5e9 s = 1024 ns (hand arithmetic).
    p = flat_profile(L=1, P=20, bw=10 ** 9)
    p["bw"][1, 11] = 2 * 10 ** 9
    assert oracle.comm_time(p, [1536], 1)[0] == 1024
    # endpoints: 2^10 at 1e9 -> 1024 ns; 2^11 at 2e9 -> 1024 ns
    assert oracle.comm_time(p, [1024, 2048], 1).tolist() == [1024, 1024]
    # quarter point: 1280 B at 1e9 + 1e9/4 = 1.25e9 -> 1024 ns
    assert oracle.comm_time(p, [1280], 1)[0] == 1024


def test_comm_time_trivial_and_ceil():
    p = flat_profile(L=2, P=12, bw=3 * 10 ** 9, lat=7)
    assert oracle.comm_time(p, [0], 1)[0] == 0          # empty transfer
    assert oracle.comm_time(p, [4096], 0)[0] == 0       # no partners
    # 1024 B at 3e9 B/s = 341.33 ns -> ceil 342, + latency 7
    assert oracle.comm_time(p, [1024], 2)[0] == 349
    assert oracle.comm_time(p, [4096], 1)[0] == 7 + math.ceil(4096e9 / 3e9)  # 2^P: bw[P]
    with pytest.raises(oracle.OracleError) as e:
        oracle.comm_time(p, [4097], 1)                  # outside the profile
    assert e.value.code == -6
    with pytest.raises(oracle.OracleError):
        oracle.comm_time(p, [1], 3)                     # group larger than the mesh


def test_comm_time_profile_points():
    # At every profiled size 2^i the time is latency + ceil(2^i*1e9 / bw[c][i])
    # exactly (interpolation endpoint): pins the choice of i (off-by-one).
    p = comm.profile(3, L=4, P=30)
    for c in range(1, 5):
        b = np.array([2 ** i for i in range(31)], np.int64)
        t = oracle.comm_time(p, b, c)
        want = [int(p["lat"][c]) + -(-(2 ** i) * 10 ** 9 // int(p["bw"][c, i])) for i in range(31)]
        assert t.tolist() == want


def test_comm_time_between_points_bracketed():
    # Monotone profile: the interpolated bandwidth lies between bw[i] and
    # bw[i+1], so the time lies between the two single-bandwidth times.
    p = comm.profile(5, L=3, P=30, monotone=True)
    rng = np.random.default_rng(1)
    b = rng.integers(1, 2 ** 30, 2000)
    for c in (1, 2, 3):
        t = oracle.comm_time(p, b, c)
        i = np.floor(np.log2(b)).astype(int)
        lo = p["bw"][c, i]
        hi = p["bw"][c, np.minimum(i + 1, 30)]
        assert np.all(t >= p["lat"][c] + np.ceil(b * 1e9 / hi) - 1)
        assert np.all(t <= p["lat"][c] + np.ceil(b * 1e9 / lo) + 1)


def test_split_states_count_and_order():
    # dims divisible by 2^L: states = compositions of <= L into D parts,
    # C(L+D, D) of them, lexicographic.
    for D, L in [(1, 3), (2, 2), (3, 4), (4, 5), (3, 6)]:
        s = oracle.split_states([2 ** L * 3] * D, L)
        assert len(s) == math.comb(L + D, D)
        assert [tuple(r) for r in s] == sorted(tuple(r) for r in s)
        assert s.sum(1).max() == L and s.min() == 0
    # divisibility: an odd dim cannot be split; dim 4 splits at most 2^2
    assert oracle.split_states([3], 3).tolist() == [[0]]
    assert oracle.split_states([4, 3], 3).tolist() == [[0, 0], [1, 0], [2, 0]]


def test_reschedule_spec_allgather():
    # SPEC.md: split [0] on mesh [4] -> replicated, shape [1024] floats: one
    # all-gather in which each device receives 4096*(4-1)/4 = 3072 bytes over
    # a group of 4, or two all-gathers over groups of 2 (1024 then 2048 B):
    # the 1-D state graph is the line (0)-(1)-(2), so these are all the paths.
    p = comm.profile(2, L=2, P=20)
    d = oracle.state_dist(p, [1024], 4)          # states (0), (1), (2)
    ct = lambda b, c: int(oracle.comm_time(p, [b], c)[0])
    assert d[2, 0] == min(ct(3072, 2), ct(1024, 1) + ct(2048, 1))
    assert d[1, 0] == ct(2048, 1)
    assert d[2, 1] == ct(1024, 1)
    assert d[0, 1] == d[0, 2] == d[1, 2] == 0   # local slices
    assert np.all(np.diag(d) == 0)


def test_reschedule_spec_dim_swap():
    # SPEC.md: split dim 0 -> split dim 1 on mesh [4], square tensor [64, 64]
    # fp32 (16384 B, shard 4096 B): one all-to-all moving the factor 4
    # (each device sends 4096 - 1024 = 3072 B over a group of 4) vs
    # gather-then-slice (each device receives 3*4096 B) vs two all-to-alls of
    # factor 2 (2048 B over groups of 2 each) -- and mixed routes, covered by
    # the brute force below.
    p = comm.profile(4, L=2, P=20)
    S = [tuple(r) for r in oracle.split_states([64, 64], 2)]
    d = oracle.state_dist(p, [64, 64], 4)
    ct = lambda b, c: int(oracle.comm_time(p, [b], c)[0])
    a, b = S.index((2, 0)), S.index((0, 2))
    direct = min(ct(3072, 2), ct(3 * 4096, 2), 2 * ct(2048, 1))
    assert d[a, b] <= direct
    assert d[a, b] == _brute(p, [64, 64], 4, 2)[a][b]


def _moves(a, dims, L, total):
    """Single collectives out of state a (R19, restated from the header text)."""
    D = len(a)
    used = sum(a)
    shard = total >> used
    ok = lambda b: sum(b) <= L and all(x >= 0 and dims[j] % (2 ** x) == 0 for j, x in enumerate(b))
    for j in range(D):
        for c in range(1, a[j] + 1):               # all-gather on dim j
            b = list(a); b[j] -= c
            yield tuple(b), ("ct", shard * (2 ** c - 1), c)
        for c in range(1, L - used + 1):           # local slice
            b = list(a); b[j] += c
            if ok(b):
                yield tuple(b), ("zero",)
        for k in range(D):                         # all-to-all j -> k
            if k == j:
                continue
            for c in range(1, a[j] + 1):
                b = list(a); b[j] -= c; b[k] += c
                if ok(b):
                    yield tuple(b), ("ct", shard - (shard >> c), c)


def _brute(p, dims, eb, L):
    """Minimum over ALL simple paths (exhaustive DFS) between every pair."""
    S = [tuple(r) for r in oracle.split_states(dims, L)]
    total = eb * int(np.prod(dims))
    w = {}
    for a in S:
        for b, m in _moves(a, dims, L, total):
            cost = 0 if m[0] == "zero" else int(oracle.comm_time(p, [m[1]], m[2])[0])
            w[(a, b)] = min(w.get((a, b), cost), cost)
    adj = {a: [(b, c) for (x, b), c in w.items() if x == a] for a in S}
    best = [[None] * len(S) for _ in S]
    for si, s in enumerate(S):
        res = {s: 0}

        def dfs(u, cost, seen):
            for v, c in adj[u]:
                if v in seen:
                    continue
                if v not in res or cost + c < res[v]:
                    res[v] = cost + c
                dfs(v, cost + c, seen | {v})
        dfs(s, 0, {s})
        best[si] = [res.get(t) for t in S]
    return best


@pytest.mark.parametrize("dims,eb,L,seed", [([64], 4, 3, 0), ([8, 12], 2, 2, 1), ([4, 4], 4, 3, 2),
                                            ([2, 6, 4], 2, 2, 3), ([16, 16], 2, 2, 4)])
def test_reschedule_bruteforce(dims, eb, L, seed):
    p = comm.profile(seed, L=L, P=24)
    d = oracle.state_dist(p, dims, eb)
    assert d.tolist() == _brute(p, dims, eb, L)


def test_reschedule_invariants():
    p = comm.profile(7, L=4, P=40)
    dims = [96, 64, 48]
    d = oracle.state_dist(p, dims, 2)
    S = [tuple(r) for r in oracle.split_states(dims, 4)]
    R = S.index((0, 0, 0))
    assert np.all(d[R] == 0)                        # replicated slices to anything for free
    assert np.all(d <= d[:, [R]] + d[[R], :])       # ... so d(a,b) <= d(a,R)
    n = len(S)
    for k in range(n):                              # triangle inequality
        assert np.all(d <= d[:, [k]] + d[[k], :])
    assert np.all(np.diag(d) == 0) and np.all(d >= 0)


def test_reschedule_costs_queries():
    p = comm.profile(8, L=3, P=40)
    nd, dims, eb = comm.tensors(8, 5, 3)
    ns = [len(oracle.split_states(dims[x, :nd[x]], 3)) for x in range(5)]
    qt, qf, qo = comm.queries(8, ns, 300)
    t = oracle.reschedule_costs(p, nd, dims, eb, qt, qf, qo)
    t2 = oracle.reschedule_costs(p, nd, dims, eb, qt, qo, qf)
    assert np.array_equal(t, t2)                    # forward + backward: symmetric
    for q in range(0, 300, 37):
        d = oracle.state_dist(p, dims[qt[q], :nd[qt[q]]], eb[qt[q]])
        assert t[q] == d[qf[q], qo[q]] + d[qo[q], qf[q]]
    assert np.all(t[qf == qo] == 0)
    with pytest.raises(oracle.OracleError):
        oracle.reschedule_costs(p, nd, dims, eb, qt[:1], np.array([999], np.int32), qo[:1])


def test_sync_costs_pins():
    # R20 (Eq. 1 m_p / t_s with P:668-671): SPEC S:231-233 examples -- fully
    # replicated on n devices: m_p = full parameter bytes; no sync partners
    # (fully split): t_s = 0 -- and the ring all-reduce volume by hand.
    p = flat_profile(L=2, P=20, bw=10 ** 9, lat=5)
    nd = np.array([1, 2], np.int32)
    dims = np.array([[1024, 1, 1, 1], [32, 64, 1, 1]], np.int64)
    eb = np.array([4, 2], np.int64)
    S0 = [tuple(r) for r in oracle.split_states([1024], 2)]     # (0), (1), (2)
    m, t = oracle.sync_costs(p, nd, dims, eb, [0, 0, 0], [S0.index((0,)), S0.index((1,)),
                                                         S0.index((2,))])
    assert m.tolist() == [4096, 2048, 1024]
    # replicated over 4: 2*(4096 - 1024) = 6144 B at 1e9 B/s -> 6144 ns + 5
    # split 2, replicated over 2: 2*(2048 - 1024) = 2048 B -> 2048 ns + 5
    assert t.tolist() == [6149, 2053, 0]
    S1 = [tuple(r) for r in oracle.split_states([32, 64], 2)]
    m, t = oracle.sync_costs(p, nd, dims, eb, [1, 1], [S1.index((1, 1)), S1.index((0, 0))])
    assert m.tolist() == [1024, 4096] and t[0] == 0 and t[1] == 6149
    with pytest.raises(oracle.OracleError):          # 2 * total > 2^P
        oracle.sync_costs(flat_profile(L=2, P=12, bw=10 ** 9), nd, dims, eb, [0], [0])
