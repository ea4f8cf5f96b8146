"""Pins for the oracle's frontier algebra (Reduce, Product, Union).

Independent of the oracle's own code: SPEC worked examples (golden file),
the pairwise Def. 1 definition, the exact left-to-right-minima distribution
(Stirling numbers of the first kind) and Lemma 2."""
import itertools
import math

import numpy as np
import pytest

import oracle
from oracle import bruteforce as bf


def test_reduce_golden(golden):
    for case in golden["reduce"]:
        inp = np.asarray(case["input"], dtype=np.int64).reshape(-1, 3)
        m, t, i = oracle.reduce(inp[:, 0], inp[:, 1], inp[:, 2].astype(np.uint64))
        got = [[int(a), int(b), int(c)] for a, b, c in zip(m, t, i)]
        assert got == case["expected"], case["id"]


def test_product_golden(golden):
    for case in golden["product"]:
        a = np.asarray(case["a"], np.int64)
        b = np.asarray(case["b"], np.int64)
        m, t, _ = oracle.segment_reduce([((a[:, 0], a[:, 1]), (b[:, 0], b[:, 1]),
                                          (np.zeros(1, np.int64), np.zeros(1, np.int64)))])
        assert [[int(x), int(y)] for x, y in zip(m, t)] == case["expected"], case["id"]


def _beats(y, x):
    """y beats x: key(y) < key(x) and t_y <= t_x (R1/R3)."""
    return (y[0], y[1], y[2]) < (x[0], x[1], x[2]) and y[1] <= x[1]


@pytest.mark.parametrize("seed", range(200))
def test_reduce_vs_pairwise_definition(seed):
    """Def. 1 pairwise: x survives iff no y beats it; heavy ties."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 60))
    hi = int(rng.choice([3, 10, 1000]))
    m = rng.integers(0, hi, n).astype(np.int64)
    t = rng.integers(0, hi, n).astype(np.int64)
    ids = rng.permutation(n).astype(np.uint64)
    pts = list(zip(m.tolist(), t.tolist(), ids.tolist()))
    want = sorted(x for x in pts if not any(_beats(y, x) for y in pts))
    fm, ft, fi = oracle.reduce(m, t, ids)
    got = list(zip(fm.tolist(), ft.tolist(), fi.tolist()))
    assert got == want
    # (m,t) set equals the id-free Def. 1 frontier
    assert [(a, b) for a, b, _ in got] == bf.pareto_def(zip(m.tolist(), t.tolist()))
    # staircase: m strictly up, t strictly down
    assert all(np.diff(fm) > 0) and all(np.diff(ft) < 0)
    # idempotent
    m2, t2, i2 = oracle.reduce(fm, ft, fi)
    assert (m2 == fm).all() and (t2 == ft).all() and (i2 == fi).all()


@pytest.mark.parametrize("seed", range(50))
def test_draft_rank_variant_equivalent(seed):
    """Draft Alg. 1 (rank by time, v = K+1) == final Alg. 1 (R2)."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 40))
    m = rng.integers(0, 6, n).astype(np.int64)
    t = rng.integers(0, 6, n).astype(np.int64)
    ids = np.arange(n, dtype=np.uint64)
    # ranks by (t, m, id), then sweep in (m, t, id) order keeping r_t < v
    order_t = sorted(range(n), key=lambda i: (t[i], m[i], ids[i]))
    rank = {i: r for r, i in enumerate(order_t)}
    v = n + 1
    keep = []
    for i in sorted(range(n), key=lambda i: (m[i], t[i], ids[i])):
        if rank[i] < v:
            keep.append(i)
            v = rank[i]
    fm, ft, fi = oracle.reduce(m, t, ids)
    assert fi.tolist() == [int(ids[i]) for i in keep]


def _stirling1(n):
    c = [[0] * (n + 1) for _ in range(n + 1)]
    c[0][0] = 1
    for i in range(1, n + 1):
        for j in range(1, i + 1):
            c[i][j] = c[i - 1][j - 1] + (i - 1) * c[i - 1][j]
    return c[n]


@pytest.mark.parametrize("K", [1, 2, 4, 6, 7])
def test_frontier_size_distribution_exact(K):
    """Assumption 1: distinct m, t a uniform permutation.  |F| is
    the number of left-to-right minima: P(|F|=j) = c(K,j)/K! (Stirling 1st
    kind), the exact form of Lemma 2.  Exhaustive over all K! orders."""
    counts = [0] * (K + 1)
    m = np.arange(K, dtype=np.int64)
    for perm in itertools.permutations(range(K)):
        fm, _, _ = oracle.reduce(m, np.asarray(perm, np.int64))
        counts[len(fm)] += 1
    assert counts == _stirling1(K)


def test_lemma2_mean_frontier_size():
    """Lemma 2: E|F| = H_K = sum 1/k.  K = 10^4, 200 trials; the
    mean lies within 3 standard errors (Var = H_K - H_K^(2))."""
    K = 10_000
    H = sum(1.0 / k for k in range(1, K + 1))
    H2 = sum(1.0 / (k * k) for k in range(1, K + 1))
    sd = math.sqrt(H - H2)
    rng = np.random.default_rng(7)
    sizes = []
    for _ in range(200):
        m = rng.permutation(K).astype(np.int64)
        t = rng.permutation(K).astype(np.int64)
        sizes.append(len(oracle.reduce(m, t)[0]))
    assert abs(np.mean(sizes) - H) < 3 * sd / math.sqrt(200)
    assert abs(H - 9.787606) < 1e-5


@pytest.mark.parametrize("seed", range(60))
def test_segment_reduce_vs_definition(seed):
    """Product + Union + Reduce with written-order ids (R6):
    the ids decode to (k, x, y, z) and re-sum to the tuple."""
    rng = np.random.default_rng(5000 + seed)
    blocks = []
    for _ in range(int(rng.integers(1, 5))):
        blk = []
        for _ in range(3):
            n = int(rng.integers(1, 5))
            blk.append((rng.integers(0, 9, n).astype(np.int64), rng.integers(0, 9, n).astype(np.int64)))
        blocks.append(blk)
    pts = []
    for k, (X, Y, Z) in enumerate(blocks):
        for x, y, z in itertools.product(range(len(X[0])), range(len(Y[0])), range(len(Z[0]))):
            pts.append((int(X[0][x] + Y[0][y] + Z[0][z]), int(X[1][x] + Y[1][y] + Z[1][z]),
                        len(pts), (k, x, y, z)))
    want = sorted(p[:3] for p in pts if not any(_beats(q[:3], p[:3]) for q in pts))
    m, t, ids = oracle.segment_reduce(blocks)
    assert list(zip(m.tolist(), t.tolist(), ids.tolist())) == want
