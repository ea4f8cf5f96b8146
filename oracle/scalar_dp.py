"""Scalar min-plus dynamic programs -- independent pins for large graphs.

TEST INFRASTRUCTURE.  These share nothing with the frontier code: they reduce
the series-parallel graph with its own (order-free) walk in a scalar
(min, +) semiring, where the optimum does not depend on elimination order:

* series  (1-in-1-out op o_i):   C_hj[w,p] = min_k C_hi[w,k] + c_i[k] + C_ij[k,p]
* parallel (edges u->v):          C[k,p]    = C1[k,p] + C2[k,p]
* K=1 source fold:                c_j[p]   += C_sj[0,p]  (+ c_s[0] once)
* chain (Viterbi):                v_i[p]    = min_k v_{i-1}[k] + C[k,p] + c_i[p]

Pins derived from them (SURVEY 8(c) "Large graphs"):

* min-memory endpoint   = lexicographic (m, t) optimum  (first frontier tuple)
* min-time endpoint     = lexicographic (t, m) optimum  (last frontier tuple)
* supported points      : min over the frontier of (b*t + a*m) = scalar optimum
  for every lambda = a/b >= 0 (the frontier contains a minimiser
  of every monotone objective).

Lexicographic costs are carried as two integer arrays (primary, secondary):
int64 while the sum of every op's and edge's largest key provably stays below
2^62, else numpy object arrays of Python ints (exact at any size: frontier
sums reach 2^60 under R10, and b*t + a*m exceeds int64 there).
"""
from __future__ import annotations

import numpy as np


def _lexmin(P, S, axis):
    """Lexicographic min over ``axis`` of pairs (P, S)."""
    pmin = P.min(axis=axis, keepdims=True)
    big = np.iinfo(np.int64).max if P.dtype == np.int64 else 1 << 200
    smin = np.where(P == pmin, S, big).min(axis=axis)
    return np.squeeze(pmin, axis=axis), smin


def solve(w, key):
    """key(m, t) -> (primary, secondary) int64 arrays; returns the optimal
    (primary, secondary) over all strategies of workload ``w``."""
    n = w.n_ops
    K = [int(k) for k in w.n_cfgs]
    op = {}
    for i in range(n):
        op[i] = key(w.op_m[i].astype(np.int64), w.op_t[i].astype(np.int64))
    edges = {}
    for e in range(w.n_edges):
        s, d = int(w.src[e]), int(w.dst[e])
        em = (np.zeros(K[s] * K[d], np.int64) if w.edge_m is None else w.edge_m[e].astype(np.int64))
        p, q = key(em, w.edge_t[e].astype(np.int64))
        edges[e] = (s, d, p.reshape(K[s], K[d]), q.reshape(K[s], K[d]))
    # exact integer type: int64 only if no partial sum can reach 2^62
    bound = sum(max(int(np.abs(a).max()), int(np.abs(b).max())) for a, b in op.values())
    bound += sum(max(int(np.abs(p).max()), int(np.abs(q).max())) for _, _, p, q in edges.values())
    if bound >= 1 << 62:
        op = {i: (a.astype(object), b.astype(object)) for i, (a, b) in op.items()}
        edges = {e: (s, d, p.astype(object), q.astype(object)) for e, (s, d, p, q) in edges.items()}
    alive = set(range(n))
    nid = w.n_edges
    # live adjacency kept incrementally (a worklist of operators and parallel
    # pairs to revisit); the scalar (min, +) optimum does not depend on the
    # order in which series / parallel / fold reductions are applied
    ins = {i: set() for i in range(n)}
    outs = {i: set() for i in range(n)}
    pairs = {}

    def link(e, s, d):
        outs[s].add(e)
        ins[d].add(e)
        pairs.setdefault((s, d), set()).add(e)

    def unlink(e):
        s, d, _, _ = edges.pop(e)
        outs[s].discard(e)
        ins[d].discard(e)
        ps = pairs[(s, d)]
        ps.discard(e)
        if not ps:
            del pairs[(s, d)]

    for e, (s, d, _, _) in edges.items():
        link(e, s, d)
    work_pairs = {k for k, v in pairs.items() if len(v) > 1}
    work_ops = set(range(n))
    while work_pairs or work_ops:
        if work_pairs:  # parallel edges: C = C1 + C2 (+ ...)
            s, d = work_pairs.pop()
            es = sorted(pairs.get((s, d), ()))
            if len(es) > 1:
                P = sum(edges[e][2] for e in es)
                Q = sum(edges[e][3] for e in es)
                for e in es:
                    unlink(e)
                edges[nid] = (s, d, P, Q)
                link(nid, s, d)
                nid += 1
                work_ops.update((s, d))
            continue
        i = work_ops.pop()
        if i not in alive:
            continue
        if len(ins[i]) == 1 and len(outs[i]) == 1:  # series: min over the middle config
            ei, eo = next(iter(ins[i])), next(iter(outs[i]))
            h, _, A, Ab = edges[ei]
            _, j, Bm, Bb = edges[eo]
            P = A[:, :, None] + op[i][0][None, :, None] + Bm[None, :, :]
            Q = Ab[:, :, None] + op[i][1][None, :, None] + Bb[None, :, :]
            Pm, Qm = _lexmin(P, Q, 1)
            unlink(ei)
            unlink(eo)
            alive.discard(i)
            edges[nid] = (h, j, Pm, Qm)
            link(nid, h, j)
            if len(pairs[(h, j)]) > 1:
                work_pairs.add((h, j))
            nid += 1
            work_ops.update((h, j))
        elif K[i] == 1 and not ins[i] and outs[i]:  # fold a K=1 source
            first = True
            for e in sorted(outs[i]):
                _, j, A, Ab = edges[e]
                p = op[j][0] + A[0]
                q = op[j][1] + Ab[0]
                if first:
                    p = p + op[i][0][0]
                    q = q + op[i][1][0]
                    first = False
                op[j] = (p, q)
                unlink(e)
                work_ops.add(j)
            alive.discard(i)
    srcs = [i for i in alive if not ins[i]]
    assert len(srcs) == 1, "scalar DP: graph is not series-parallel reducible"
    cur = srcs[0]
    vP, vQ = op[cur]
    seen = 1
    while outs[cur]:
        assert len(outs[cur]) == 1
        _, j, A, Ab = edges[next(iter(outs[cur]))]
        P = vP[:, None] + A
        Q = vQ[:, None] + Ab
        pm, qm = _lexmin(P, Q, 0)
        vP = pm + op[j][0]
        vQ = qm + op[j][1]
        cur = j
        seen += 1
    assert seen == len(alive)
    best = _lexmin(vP[:, None], vQ[:, None], 0)
    return int(best[0][0]), int(best[1][0])


def min_memory_endpoint(w):
    """(m, t) of the lexicographically smallest (m, t) strategy."""
    return solve(w, lambda m, t: (m, t))


def min_time_endpoint(w):
    """(m, t) of the lexicographically smallest (t, m) strategy."""
    t, m = solve(w, lambda m, t: (t, m))
    return m, t


def weighted_optimum(w, a: int, b: int):
    """min over strategies of b*t + a*m (exact; a, b non-negative ints)."""
    if max(a, b) < 1 << 20:  # per-entry keys fit int64 (costs < 2^40, R10); solve() widens sums
        z = lambda m, t: (b * t + a * m, np.zeros_like(m))
    else:
        z = lambda m, t: (b * t.astype(object) + a * m.astype(object), np.zeros(len(m), np.int64))
    return solve(w, z)[0]


def min_memory_closed_form(w):
    """Sum over ops of min_k m(o_i, k) (valid when every edge m is 0, Eq. 2)."""
    assert w.edge_m is None
    return int(sum(int(x.min()) for x in w.op_m))
