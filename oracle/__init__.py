"""CPU oracle for the FT hot path (arXiv 2004.10856) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA product path (``paper_2004_10856_b200``); the
only common module is the seeded input generator ``synth``.

* ``liboracle_ft.so`` (``oracle_ft.cpp``): plain C++17 step algorithm of
  SURVEY 8(c) -- Alg. 1 reduce, Product/Union, Eq. 4, Eq. 5, K=1 Eq. 7, Alg. 3
  LDP, unroll -- the bit-exact target of the GPU path.
* ``bruteforce.py``: pure-Python Eq. 3 enumeration + definition-level
  Pareto filter (Def. 1) for tiny graphs.
* ``scalar_dp.py``: scalar min-plus DPs (endpoints, supported points) for
  graphs too large for brute force.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_ft.so")

OK, EINVAL, ESTATE, EPRECOND, ENOMEM, EOVERFLOW, ESIZE, EINTERNAL = 0, -1, -2, -3, -4, -6, -7, -8
NODE, EDGE, AUTO, AUTO_HEUR = 1, 2, 3, 4
STEP_NAMES = {1: "node", 2: "edge", 3: "fold", 4: "ldp", 5: "final", 6: "pair", 7: "branch", 8: "compose",
              9: "remap"}


def build(force: bool = False) -> str:
    """Compile liboracle_ft.so with g++ (plain -O2, no vectorisation tricks)."""
    srcs = [os.path.join(_HERE, f) for f in ("oracle_ft.cpp", "oracle_costgen.cpp")]
    hdr = os.path.join(_HERE, "oracle_ft.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(f) for f in srcs + [hdr])):
        return LIB_PATH
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-Wall", "-shared", "-fPIC", "-o",
                           LIB_PATH, *srcs, "-lpthread"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P64 = C.POINTER(C.c_int64)
        PU64 = C.POINTER(C.c_uint64)
        P32 = C.POINTER(C.c_int32)
        L.oft_graph_create.argtypes = [C.c_int32, P32, C.c_int32, P32, P32, C.c_int32,
                                       C.POINTER(C.c_void_p)]
        L.oft_graph_destroy.argtypes = [C.c_void_p]
        L.oft_set_op_costs.argtypes = [C.c_void_p, C.c_int32, P64, P64]
        L.oft_set_edge_costs.argtypes = [C.c_void_p, C.c_int32, P64, P64]
        L.oft_eliminate.argtypes = [C.c_void_p, C.c_int32, C.c_int32, P32]
        L.oft_frontier.argtypes = [C.c_void_p, C.c_int64, P64, P64, P64]
        L.oft_frontier_elim.argtypes = [C.c_void_p, C.c_int64, P64, P64, P64]
        L.oft_query_mini_time.argtypes = [C.c_void_p, C.c_int64, P64]
        L.oft_strategy.argtypes = [C.c_void_p, C.c_int64, P32]
        L.oft_set_heuristic.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64]
        L.oft_num_steps.argtypes = [C.c_void_p]
        L.oft_num_steps.restype = C.c_int64
        L.oft_step_info.argtypes = [C.c_void_p, C.c_int64, P64]
        L.oft_step_output.argtypes = [C.c_void_p, C.c_int64, C.c_int64, P64, P64, P64, PU64]
        L.oft_last_error.argtypes = [C.c_void_p]
        L.oft_last_error.restype = C.c_char_p
        L.oft_reduce.argtypes = [C.c_int64, P64, P64, PU64, P64, P64, PU64, P64]
        L.oft_segment_reduce.argtypes = [C.c_int32] + [P64] * 9 + [C.c_int64, P64, P64, PU64, P64]
        L.ocg_comm_time.argtypes = [C.c_void_p, C.c_int64, P64, P32, P64]
        L.ocg_split_states.argtypes = [C.c_int32, P64, C.c_int32, C.c_int64, P32, P64]
        L.ocg_state_dist.argtypes = [C.c_void_p, C.c_int32, P64, C.c_int64, C.c_int64, P64, P64]
        L.ocg_sync_costs.argtypes = [C.c_void_p, C.c_int32, P32, P64, P64, C.c_int64, P32, P32,
                                     P64, P64]
        L.ocg_reschedule_costs.argtypes = [C.c_void_p, C.c_int32, P32, P64, P64, C.c_int64,
                                           P32, P32, P32, P64]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


class Graph:
    """ctypes handle over liboracle_ft.so with the same call sequence as the
    product binding (create, set costs, eliminate, frontier, strategy)."""

    def __init__(self, n_cfgs, src, dst, threads: int = 1):
        L = lib()
        self._L = L
        n_cfgs = np.ascontiguousarray(n_cfgs, dtype=np.int32)
        src = np.ascontiguousarray(src, dtype=np.int32)
        dst = np.ascontiguousarray(dst, dtype=np.int32)
        self.n_ops = len(n_cfgs)
        self.K = n_cfgs
        h = C.c_void_p()
        rc = L.oft_graph_create(self.n_ops, _p(n_cfgs, C.c_int32), len(src), _p(src, C.c_int32),
                                _p(dst, C.c_int32), int(threads), C.byref(h))
        if rc:
            raise OracleError(rc, "graph_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self._L.oft_graph_destroy(self.h)
            self.h = None

    __del__ = close

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self._L.oft_last_error(self.h).decode())
        return rc

    def set_op_costs(self, op, m, t):
        m = np.ascontiguousarray(m, dtype=np.int64)
        t = np.ascontiguousarray(t, dtype=np.int64)
        return self._chk(self._L.oft_set_op_costs(self.h, op, _p(m, C.c_int64), _p(t, C.c_int64)))

    def set_edge_costs(self, e, m, t):
        t = np.ascontiguousarray(t, dtype=np.int64)
        if m is not None:
            m = np.ascontiguousarray(m, dtype=np.int64)
        return self._chk(self._L.oft_set_edge_costs(self.h, e, _p(m, C.c_int64), _p(t, C.c_int64)))

    def eliminate(self, kind=AUTO, id=-1):
        ne = C.c_int32(-1)
        self._chk(self._L.oft_eliminate(self.h, kind, id, C.byref(ne)))
        return ne.value

    def frontier(self, algo="ldp"):
        """Final frontier by FT-LDP (Alg. 3) or, algo="elim", FT-Elimination."""
        fn = self._L.oft_frontier if algo == "ldp" else self._L.oft_frontier_elim
        n = C.c_int64(0)
        rc = fn(self.h, 0, None, None, C.byref(n))
        if rc not in (OK, ESIZE):
            self._chk(rc)
        m = np.empty(n.value, np.int64)
        t = np.empty(n.value, np.int64)
        self._chk(fn(self.h, n.value, _p(m, C.c_int64), _p(t, C.c_int64), C.byref(n)))
        return m, t

    def set_heuristic(self, policy="min_memory", alpha=(1, 2)):
        """Heuristic-elimination rule: "min_memory" (R17) or "weighted"
        alpha*m/M + (1-alpha)*t/T, alpha = num/den (R22)."""
        pol = {"min_memory": 0, "weighted": 1}[policy]
        return self._chk(self._L.oft_set_heuristic(self.h, pol, int(alpha[0]), int(alpha[1])))

    def mini_time(self, memory_limit):
        """SS4.1 mini-time: index of the fastest frontier tuple with m <= limit, or -1."""
        i = C.c_int64(-1)
        self._chk(self._L.oft_query_mini_time(self.h, int(memory_limit), C.byref(i)))
        return i.value

    def strategy(self, idx):
        out = np.empty(self.n_ops, np.int32)
        self._chk(self._L.oft_strategy(self.h, idx, _p(out, C.c_int32)))
        return out

    def num_steps(self):
        return int(self._L.oft_num_steps(self.h))

    def step_info(self, s):
        info = np.empty(6, np.int64)
        self._chk(self._L.oft_step_info(self.h, s, _p(info, C.c_int64)))
        return {"kind": STEP_NAMES[int(info[0])], "nseg": int(info[1]), "nblk": int(info[2]),
                "tuples": int(info[3]), "survivors": int(info[4]), "us": int(info[5])}

    def step_output(self, s):
        info = self.step_info(s)
        n = info["survivors"]
        so = np.empty(info["nseg"] + 1, np.int64)
        m = np.empty(n, np.int64)
        t = np.empty(n, np.int64)
        bp = np.empty(n, np.uint64)
        self._chk(self._L.oft_step_output(self.h, s, n, _p(so, C.c_int64), _p(m, C.c_int64),
                                          _p(t, C.c_int64), _p(bp, C.c_uint64)))
        return so, m, t, bp


def load(w, threads: int = 1) -> Graph:
    """Create an oracle graph from a ``synth.graphs.Workload`` and set its costs."""
    g = Graph(w.n_cfgs, w.src, w.dst, threads)
    for i in range(w.n_ops):
        g.set_op_costs(i, w.op_m[i], w.op_t[i])
    for e in range(w.n_edges):
        g.set_edge_costs(e, None if w.edge_m is None else w.edge_m[e], w.edge_t[e])
    return g


def run_ft(w, threads: int = 1):
    """FT_AUTO + LDP on a workload; returns (graph, m, t)."""
    g = load(w, threads)
    g.eliminate(AUTO)
    m, t = g.frontier()
    return g, m, t


def reduce(m, t, ids=None):
    """Alg. 1 on an explicit list; returns (m, t, id) of the frontier."""
    m = np.ascontiguousarray(m, dtype=np.int64)
    t = np.ascontiguousarray(t, dtype=np.int64)
    n = len(m)
    ids = None if ids is None else np.ascontiguousarray(ids, dtype=np.uint64)
    mo = np.empty(n, np.int64)
    to = np.empty(n, np.int64)
    io = np.empty(n, np.uint64)
    no = C.c_int64(0)
    rc = lib().oft_reduce(n, _p(m, C.c_int64), _p(t, C.c_int64), _p(ids, C.c_uint64),
                          _p(mo, C.c_int64), _p(to, C.c_int64), _p(io, C.c_uint64), C.byref(no))
    if rc:
        raise OracleError(rc, "reduce")
    k = no.value
    return mo[:k], to[:k], io[:k]


def segment_reduce(blocks):
    """blocks: list of (X, Y, Z) with each factor a pair (m[], t[]).  Returns
    (m, t, id) = reduce(U_k X_k (x) Y_k (x) Z_k) with written-order ids."""
    def cat(idx):
        offs = [0]
        ms, ts = [], []
        for b in blocks:
            mm, tt = b[idx]
            ms.append(np.asarray(mm, np.int64))
            ts.append(np.asarray(tt, np.int64))
            offs.append(offs[-1] + len(mm))
        return (np.asarray(offs, np.int64),
                np.ascontiguousarray(np.concatenate(ms) if ms else np.zeros(0, np.int64)),
                np.ascontiguousarray(np.concatenate(ts) if ts else np.zeros(0, np.int64)))
    xs, ys, zs = cat(0), cat(1), cat(2)
    total = sum(len(b[0][0]) * len(b[1][0]) * len(b[2][0]) for b in blocks)
    cap = max(total, 1)
    mo = np.empty(cap, np.int64)
    to = np.empty(cap, np.int64)
    io = np.empty(cap, np.uint64)
    no = C.c_int64(0)
    args = []
    for (o, mm, tt) in (xs, ys, zs):
        args += [_p(o, C.c_int64), _p(mm, C.c_int64), _p(tt, C.c_int64)]
    rc = lib().oft_segment_reduce(len(blocks), *args, cap, _p(mo, C.c_int64), _p(to, C.c_int64),
                                  _p(io, C.c_uint64), C.byref(no))
    if rc:
        raise OracleError(rc, "segment_reduce")
    k = no.value
    return mo[:k], to[:k], io[:k]


# ---------------------------------------------------------------------------
# Edge-cost generation (oracle_costgen.cpp)
# ---------------------------------------------------------------------------
class _Profile(C.Structure):
    _fields_ = [("L", C.c_int32), ("P", C.c_int32), ("lat", C.c_int64 * 7),
                ("bw", (C.c_int64 * 47) * 7)]


def _profile(prof) -> _Profile:
    p = _Profile()
    p.L, p.P = int(prof["L"]), int(prof["P"])
    for c in range(7):
        p.lat[c] = int(prof["lat"][c])
        for i in range(47):
            p.bw[c][i] = int(prof["bw"][c][i])
    return p


def _check(rc, what):
    if rc != 0:
        raise OracleError(rc, what)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what}: error {code}")
        self.code = code


def comm_time(prof, nbytes, group_log2) -> np.ndarray:
    """P:668-671 interpolated communication time in ns (R18)."""
    b = np.ascontiguousarray(nbytes, np.int64)
    g = np.ascontiguousarray(np.broadcast_to(np.asarray(group_log2, np.int32), b.shape), np.int32)
    out = np.zeros(b.shape, np.int64)
    p = _profile(prof)
    _check(lib().ocg_comm_time(C.byref(p), b.size, _p(b, C.c_int64), _p(g, C.c_int32),
                               _p(out, C.c_int64)), "comm_time")
    return out


def split_states(dims, L: int) -> np.ndarray:
    """Split states (R19) of a tensor with shape `dims` on 2^L devices, [S, D] int32."""
    d = np.ascontiguousarray(dims, np.int64)
    n = C.c_int64(0)
    rc = lib().ocg_split_states(d.size, _p(d, C.c_int64), L, 0, None, C.byref(n))
    out = np.zeros((n.value, d.size), np.int32)
    _check(lib().ocg_split_states(d.size, _p(d, C.c_int64), L, n.value, _p(out, C.c_int32),
                                  C.byref(n)), "split_states")
    return out


def state_dist(prof, dims, elem_bytes: int) -> np.ndarray:
    """All-pairs re-scheduling distances (Dijkstra), [S, S] int64."""
    d = np.ascontiguousarray(dims, np.int64)
    S = len(split_states(d, int(prof["L"])))
    out = np.zeros((S, S), np.int64)
    n = C.c_int64(0)
    p = _profile(prof)
    _check(lib().ocg_state_dist(C.byref(p), d.size, _p(d, C.c_int64), int(elem_bytes), S * S,
                                _p(out, C.c_int64), C.byref(n)), "state_dist")
    return out


def reschedule_costs(prof, ndims, dims, elem_bytes, q_tensor, q_from, q_to) -> np.ndarray:
    """t_x = d(from,to) + d(to,from) per query (Eq. 2 + P:860, R19)."""
    nd = np.ascontiguousarray(ndims, np.int32)
    dm = np.ascontiguousarray(dims, np.int64)
    eb = np.ascontiguousarray(elem_bytes, np.int64)
    qt, qf, qo = (np.ascontiguousarray(a, np.int32) for a in (q_tensor, q_from, q_to))
    out = np.zeros(qt.size, np.int64)
    p = _profile(prof)
    _check(lib().ocg_reschedule_costs(C.byref(p), nd.size, _p(nd, C.c_int32), _p(dm, C.c_int64),
                                      _p(eb, C.c_int64), qt.size, _p(qt, C.c_int32),
                                      _p(qf, C.c_int32), _p(qo, C.c_int32), _p(out, C.c_int64)),
           "reschedule_costs")
    return out


def sync_costs(prof, ndims, dims, elem_bytes, q_tensor, q_state):
    """(m_p, t_s) of a parameter tensor in a split state (Eq. 1 + P:668-671, R20)."""
    nd = np.ascontiguousarray(ndims, np.int32)
    dm = np.ascontiguousarray(dims, np.int64)
    eb = np.ascontiguousarray(elem_bytes, np.int64)
    qt, qs = (np.ascontiguousarray(a, np.int32) for a in (q_tensor, q_state))
    m = np.zeros(qt.size, np.int64)
    t = np.zeros(qt.size, np.int64)
    p = _profile(prof)
    _check(lib().ocg_sync_costs(C.byref(p), nd.size, _p(nd, C.c_int32), _p(dm, C.c_int64),
                                _p(eb, C.c_int64), qt.size, _p(qt, C.c_int32), _p(qs, C.c_int32),
                                _p(m, C.c_int64), _p(t, C.c_int64)), "sync_costs")
    return m, t
