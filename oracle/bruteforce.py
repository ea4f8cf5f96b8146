"""Brute force over all strategies -- TEST INFRASTRUCTURE.

Plain definitions, no FT machinery:

* ``total_cost``  -- Eq. 3: t(S) = sum of op t + sum of edge t,
  m(S) = sum of op m (+ edge m when given; 0 by Eq. 2).
* ``pareto_def``  -- Def. 1 written out pairwise, O(n^2): the
  minimum subset F such that every tuple is dominated-or-equalled by one in F.
* ``enumerate_costs`` -- all prod(K_i) strategies, vectorised Eq. 3.
* ``check_frontier`` -- Def. 1 checked against the full enumeration without
  sorting: every F point is achieved, no enumerated point strictly dominates
  an F point, every enumerated point is weakly dominated by an F point, and F
  is duplicate-free and mutually non-dominated.
"""
from __future__ import annotations

import itertools

import numpy as np


def total_cost(w, S):
    """Eq. 3 for one full strategy S (config index per op)."""
    m = 0
    t = 0
    for i in range(w.n_ops):
        m += int(w.op_m[i][S[i]])
        t += int(w.op_t[i][S[i]])
    for e in range(w.n_edges):
        s, d = int(w.src[e]), int(w.dst[e])
        k = int(S[s]) * int(w.n_cfgs[d]) + int(S[d])
        t += int(w.edge_t[e][k])
        if w.edge_m is not None:
            m += int(w.edge_m[e][k])
    return m, t


def pareto_def(points):
    """Def. 1 pairwise: keep p iff no q with q.m <= p.m, q.t <= p.t and
    (q.m, q.t) != (p.m, p.t); duplicates collapse to one (m, t)."""
    pts = sorted(set((int(a), int(b)) for a, b in points))
    out = []
    for p in pts:
        dominated = False
        for q in pts:
            if q != p and q[0] <= p[0] and q[1] <= p[1]:
                dominated = True
                break
        if not dominated:
            out.append(p)
    return out


def enumerate_costs(w, limit: int = 2_000_000):
    """(m[], t[], cfg[N, n_ops]) over all prod(K_i) strategies (mixed radix,
    op 0 most significant)."""
    K = [int(k) for k in w.n_cfgs]
    total = 1
    for k in K:
        total *= k
    if total > limit:
        raise ValueError(f"{total} strategies > limit {limit}")
    idx = np.arange(total, dtype=np.int64)
    cfg = np.empty((total, w.n_ops), dtype=np.int64)
    stride = total
    for i, k in enumerate(K):
        stride //= k
        cfg[:, i] = (idx // stride) % k
    m = np.zeros(total, np.int64)
    t = np.zeros(total, np.int64)
    for i in range(w.n_ops):
        m += w.op_m[i][cfg[:, i]]
        t += w.op_t[i][cfg[:, i]]
    for e in range(w.n_edges):
        s, d = int(w.src[e]), int(w.dst[e])
        k = cfg[:, s] * K[d] + cfg[:, d]
        t += w.edge_t[e][k]
        if w.edge_m is not None:
            m += w.edge_m[e][k]
    return m, t, cfg


def brute_force(w, limit: int = 200_000):
    """Definition-level frontier (sorted by m) of all strategies, small cases."""
    m, t, _ = enumerate_costs(w, limit)
    return pareto_def(zip(m.tolist(), t.tolist()))


def check_frontier(fm, ft, m_all, t_all):
    """Def. 1 against a full enumeration; returns a list of violations."""
    bad = []
    fm = np.asarray(fm, np.int64)
    ft = np.asarray(ft, np.int64)
    pts = set(zip(m_all.tolist(), t_all.tolist()))
    if len(set(zip(fm.tolist(), ft.tolist()))) != len(fm):
        bad.append("duplicate (m,t) in frontier")
    for a, b in zip(fm.tolist(), ft.tolist()):
        if (a, b) not in pts:
            bad.append(f"frontier point {(a, b)} not achieved by any strategy")
        strict = (m_all <= a) & (t_all <= b) & ((m_all < a) | (t_all < b))
        if strict.any():
            bad.append(f"frontier point {(a, b)} strictly dominated")
    # every enumerated point weakly dominated by some frontier point (chunked O(N*F))
    for lo in range(0, len(m_all), 65536):
        mm = m_all[lo:lo + 65536, None]
        tt = t_all[lo:lo + 65536, None]
        cover = ((fm[None, :] <= mm) & (ft[None, :] <= tt)).any(axis=1)
        if not cover.all():
            j = int(np.argmin(cover))
            bad.append(f"point {(int(mm[j, 0]), int(tt[j, 0]))} not covered")
            break
    return bad


def all_strategies(w):
    return itertools.product(*[range(int(k)) for k in w.n_cfgs])
