"""paper_2004_10856_b200 -- B200-native Frontier Tracking (arXiv 2004.10856).

Thin ctypes binding over ``libft.so`` (C-ABI: ``include/ft.h``).  Argument
marshalling only: every step of the FT hot path (Product / Union / Reduce of
every node elimination, edge elimination, K=1 fold, LDP step and final
reduce) runs in the sm_100a kernels of ``csrc/``.  There is no CPU fallback:
if the library cannot be loaded, importing this package raises.

Same names as the C-ABI:

    g = Graph(n_cfgs, src, dst)           # ft_graph_create
    g.set_op_costs(op, m, t)              # ft_set_op_costs   (Eq. 1)
    g.set_edge_costs(e, m, t)             # ft_set_edge_costs (Eq. 2)
    g.eliminate(AUTO)                     # ft_eliminate      (Alg. 2 lines 4-11)
    m, t = g.frontier()                   # ft_frontier       (Alg. 3)
    cfg = g.strategy(i)                   # ft_strategy       (unroll)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libft.so")

OK, EINVAL, ESTATE, EPRECOND, ENOMEM, ECUDA, EOVERFLOW, ESIZE, EINTERNAL = 0, -1, -2, -3, -4, -5, -6, -7, -8
NODE, EDGE, AUTO, AUTO_HEUR = 1, 2, 3, 4
STEP_KINDS = {1: "node", 2: "edge", 3: "fold", 4: "ldp", 5: "final", 6: "pair", 7: "branch", 8: "compose",
              9: "remap"}


class FTError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libft error {code}: {msg}")
        self.code = code


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class ft_options(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", C.c_void_p), ("rank", C.c_int32),
                ("world", C.c_int32), ("nccl_comm", C.c_void_p), ("keep_all", C.c_int32),
                ("profile", C.c_int32), ("loopback", C.c_int32), ("alloc", C.c_void_p),
                ("free", C.c_void_p), ("alloc_ctx", C.c_void_p), ("reserved", C.c_int32 * 4)]


class ft_step_stats(C.Structure):
    _fields_ = [("kind", C.c_int32), ("levels", C.c_int32), ("wave", C.c_int32),
                ("pad", C.c_int32), ("nseg", C.c_int64),
                ("nblk", C.c_int64), ("tuples", C.c_int64), ("survivors", C.c_int64),
                ("candidates", C.c_int64), ("retries", C.c_int64), ("launches", C.c_int64),
                ("max_seg", C.c_int64), ("filter_tuples", C.c_int64), ("direct_tuples", C.c_int64),
                ("kernel_ms", C.c_float), ("comm_ms", C.c_float), ("plan_ms", C.c_float),
                ("direct_ms", C.c_float), ("filter_ms", C.c_float), ("bucket_ms", C.c_float),
                ("compact_ms", C.c_float), ("host_ms", C.c_float), ("path", C.c_int64 * 4)]


CG_MAX_MESH, CG_MAX_P, CG_MAX_DIMS = 6, 46, 4


class ft_comm_profile(C.Structure):
    _fields_ = [("mesh_log2", C.c_int32), ("P", C.c_int32),
                ("latency_ns", C.c_int64 * (CG_MAX_MESH + 1)),
                ("bw", (C.c_int64 * (CG_MAX_P + 1)) * (CG_MAX_MESH + 1))]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libft.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P64, PU64, P32 = C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.POINTER(C.c_int32)
    L.ft_graph_create.argtypes = [C.c_int32, P32, C.c_int32, P32, P32, C.POINTER(ft_options),
                                  C.POINTER(C.c_void_p)]
    L.ft_graph_destroy.argtypes = [C.c_void_p]
    L.ft_graph_destroy.restype = None
    L.ft_set_op_costs.argtypes = [C.c_void_p, C.c_int32, P64, P64]
    L.ft_set_edge_costs.argtypes = [C.c_void_p, C.c_int32, P64, P64]
    L.ft_eliminate.argtypes = [C.c_void_p, C.c_int32, C.c_int32, P32]
    L.ft_frontier.argtypes = [C.c_void_p, C.c_int64, P64, P64, P64]
    L.ft_frontier_elim.argtypes = [C.c_void_p, C.c_int64, P64, P64, P64]
    L.ft_query_mini_time.argtypes = [C.c_void_p, C.c_int64, P64]
    L.ft_strategy.argtypes = [C.c_void_p, C.c_int64, P32]
    L.ft_set_heuristic.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64]
    L.ft_get_stats.argtypes = [C.c_void_p, C.POINTER(ft_step_stats), C.c_int64, P64]
    L.ft_step_output.argtypes = [C.c_void_p, C.c_int64, C.c_int64, P64, P64, P64, PU64, P64]
    L.ft_shard_plan.argtypes = [C.c_int64, P64, C.c_int32, P64]
    L.ft_prepare.argtypes = [C.c_void_p]
    L.ft_set_costs_all.argtypes = [C.c_void_p, P64, P64, P64, P64]
    L.ft_step_inputs.argtypes = [C.c_void_p, C.c_int64, P64, P64]
    L.ft_nccl_unique_id.argtypes = [C.c_char_p]
    L.ft_nccl_comm_init.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.c_int32,
                                    C.POINTER(C.c_void_p)]
    L.ft_nccl_comm_destroy.argtypes = [C.c_void_p]
    L.ft_last_error.argtypes = [C.c_void_p]
    L.ft_last_error.restype = C.c_char_p
    L.ft_version.argtypes = []
    L.ft_version.restype = C.c_char_p
    L.ft_comm_time.argtypes = [C.POINTER(ft_comm_profile), C.c_int64, P64, P32, P64]
    L.ft_split_states.argtypes = [C.c_int32, P64, C.c_int32, C.c_int64, P32, P64]
    L.ft_reschedule_costs.argtypes = [C.POINTER(ft_comm_profile), C.c_int32, P32, P64, P64,
                                      C.c_int64, P32, P32, P32, P64]
    L.ft_sync_costs.argtypes = [C.POINTER(ft_comm_profile), C.c_int32, P32, P64, P64, C.c_int64,
                                P32, P32, P64, P64]
    L.ft_costgen_profile.argtypes = [C.c_int32]
    L.ft_costgen_last_times.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float)]
    L.ft_reschedule_costs_dev.argtypes = [C.POINTER(ft_comm_profile), C.c_int32, P32, P64, P64,
                                          C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
    return L


lib = _load()
TORCH_ALLOC_PATH = os.path.join(_HERE, "libft_torch_alloc.so")
_torch_alloc = None


def torch_allocator():
    """(alloc, free) C function pointers backed by torch's CUDA caching
    allocator (libft_torch_alloc.so, csrc/ft_torch_alloc.cpp) for
    ft_options.alloc / .free: no Python on the allocation path."""
    global _torch_alloc
    if _torch_alloc is None:
        import torch  # noqa: F401  (libc10_cuda must be loaded and initialised)
        torch.cuda.init()
        if not os.path.exists(TORCH_ALLOC_PATH):
            raise ImportError(f"{TORCH_ALLOC_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(TORCH_ALLOC_PATH)
        _torch_alloc = (L, C.cast(L.ft_torch_alloc, C.c_void_p).value, C.cast(L.ft_torch_free, C.c_void_p).value)
    return _torch_alloc[1], _torch_alloc[2]
SYMBOLS = ["ft_graph_create", "ft_graph_destroy", "ft_set_op_costs", "ft_set_edge_costs",
           "ft_eliminate", "ft_frontier", "ft_set_heuristic", "ft_frontier_elim", "ft_query_mini_time", "ft_strategy", "ft_get_stats", "ft_step_output",
           "ft_prepare", "ft_set_costs_all", "ft_step_inputs", "ft_shard_plan", "ft_nccl_unique_id",
           "ft_nccl_comm_init", "ft_nccl_comm_destroy", "ft_last_error", "ft_version",
           "ft_comm_time", "ft_split_states", "ft_reschedule_costs", "ft_reschedule_costs_dev", "ft_sync_costs", "ft_costgen_profile",
           "ft_costgen_last_times"]


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def shard_plan(weights, world: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, dtype=np.int64)
    b = np.zeros(world + 1, np.int64)
    rc = lib.ft_shard_plan(len(w), _p(w, C.c_int64), world, _p(b, C.c_int64))
    if rc:
        raise FTError(rc, "shard_plan")
    return b


class Graph:
    def __init__(self, n_cfgs, src, dst, device: int = 0, stream=None, rank: int = 0,
                 world: int = 1, nccl_comm=None, keep_all: bool = False, profile: bool = False,
                 loopback: bool = False, torch_alloc: bool = False, alloc=None):
        """alloc: optional (alloc_fn, free_fn[, ctx]) raw C function pointers
        (ints) for ft_options.alloc / .free; torch_alloc=True uses torch's
        caching allocator (torch_allocator())."""
        K = np.ascontiguousarray(n_cfgs, dtype=np.int32)
        s = np.ascontiguousarray(src, dtype=np.int32)
        d = np.ascontiguousarray(dst, dtype=np.int32)
        self.n_ops = len(K)
        opt = ft_options()
        opt.device = device
        opt.stream = stream
        opt.rank = rank
        opt.world = world
        opt.nccl_comm = nccl_comm
        opt.keep_all = 1 if keep_all else 0
        opt.profile = 1 if profile else 0
        opt.loopback = 1 if loopback else 0
        if torch_alloc and alloc is None:
            alloc = torch_allocator()
        if alloc is not None:
            opt.alloc = alloc[0]
            opt.free = alloc[1]
            opt.alloc_ctx = alloc[2] if len(alloc) > 2 else None
        h = C.c_void_p()
        rc = lib.ft_graph_create(self.n_ops, _p(K, C.c_int32), len(s), _p(s, C.c_int32),
                                 _p(d, C.c_int32), C.byref(opt), C.byref(h))
        if rc:
            raise FTError(rc, "ft_graph_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib.ft_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        if rc:
            raise FTError(rc, lib.ft_last_error(self.h).decode())

    def set_op_costs(self, op, m, t):
        m = np.ascontiguousarray(m, dtype=np.int64)
        t = np.ascontiguousarray(t, dtype=np.int64)
        self._chk(lib.ft_set_op_costs(self.h, op, _p(m, C.c_int64), _p(t, C.c_int64)))

    def set_edge_costs(self, e, m, t):
        t = np.ascontiguousarray(t, dtype=np.int64)
        m = None if m is None else np.ascontiguousarray(m, dtype=np.int64)
        self._chk(lib.ft_set_edge_costs(self.h, e, _p(m, C.c_int64), _p(t, C.c_int64)))

    def set_costs_all(self, op_m, op_t, edge_m, edge_t):
        """Concatenated cost arrays (see ft_set_costs_all); pinned numpy views
        (e.g. torch.empty(..., pin_memory=True).numpy()) give the fastest copy."""
        op_m = np.ascontiguousarray(op_m, dtype=np.int64)
        op_t = np.ascontiguousarray(op_t, dtype=np.int64)
        edge_t = np.ascontiguousarray(edge_t, dtype=np.int64)
        edge_m = None if edge_m is None else np.ascontiguousarray(edge_m, dtype=np.int64)
        self._chk(lib.ft_set_costs_all(self.h, _p(op_m, C.c_int64), _p(op_t, C.c_int64),
                                       _p(edge_m, C.c_int64), _p(edge_t, C.c_int64)))

    def prepare(self):
        self._chk(lib.ft_prepare(self.h))

    def step_inputs(self, step: int):
        src = np.zeros(6, np.int64)
        par = np.zeros(6, np.int64)
        self._chk(lib.ft_step_inputs(self.h, step, _p(src, C.c_int64), _p(par, C.c_int64)))
        return src.reshape(3, 2), par

    def eliminate(self, kind: int = AUTO, id: int = -1) -> int:
        ne = C.c_int32(-1)
        self._chk(lib.ft_eliminate(self.h, kind, id, C.byref(ne)))
        return ne.value

    def frontier(self, algo: str = "ldp"):
        """Final frontier by FT-LDP (Alg. 3, ft_frontier) or, with algo="elim",
        FT-Elimination (ft_frontier_elim)."""
        fn = lib.ft_frontier if algo == "ldp" else lib.ft_frontier_elim
        n = C.c_int64(0)
        rc = fn(self.h, 0, None, None, C.byref(n))
        if rc not in (OK, ESIZE):
            self._chk(rc)
        m = np.empty(n.value, np.int64)
        t = np.empty(n.value, np.int64)
        self._chk(fn(self.h, n.value, _p(m, C.c_int64), _p(t, C.c_int64), C.byref(n)))
        return m, t

    def set_heuristic(self, policy: str = "min_memory", alpha=(1, 2)):
        """ft_set_heuristic: "min_memory" (R17) or "weighted" alpha*m/M +
        (1-alpha)*t/T with alpha = num/den (R22)."""
        pol = {"min_memory": 0, "weighted": 1}[policy]
        self._chk(lib.ft_set_heuristic(self.h, pol, int(alpha[0]), int(alpha[1])))

    def mini_time(self, memory_limit: int) -> int:
        """SS4.1 mini-time: index of the fastest frontier tuple with m <= limit, or -1."""
        i = C.c_int64(-1)
        self._chk(lib.ft_query_mini_time(self.h, int(memory_limit), C.byref(i)))
        return i.value

    def strategy(self, idx: int) -> np.ndarray:
        out = np.empty(self.n_ops, np.int32)
        self._chk(lib.ft_strategy(self.h, int(idx), _p(out, C.c_int32)))
        return out

    def stats(self):
        n = C.c_int64(0)
        lib.ft_get_stats(self.h, None, 0, C.byref(n))
        buf = (ft_step_stats * max(1, n.value))()
        self._chk(lib.ft_get_stats(self.h, buf, n.value, C.byref(n)))
        out = []
        for i in range(n.value):
            s = buf[i]
            out.append({"kind": STEP_KINDS.get(s.kind, s.kind), "levels": s.levels, "wave": s.wave,
                        "nseg": s.nseg,
                        "nblk": s.nblk, "tuples": s.tuples, "survivors": s.survivors,
                        "candidates": s.candidates, "retries": s.retries,
                        "launches": s.launches, "kernel_ms": s.kernel_ms, "comm_ms": s.comm_ms,
                        "plan_ms": s.plan_ms, "direct_ms": s.direct_ms, "filter_ms": s.filter_ms,
                        "bucket_ms": s.bucket_ms, "compact_ms": s.compact_ms,
                        "host_ms": s.host_ms, "max_seg": s.max_seg,
                        "filter_tuples": s.filter_tuples, "direct_tuples": s.direct_tuples,
                        "path": {"shared_rows": s.path[0], "shared_tie_rows": s.path[1],
                                 "shared_cta_rows": s.path[2], "direct_reg_segs": s.path[3]}})
        return out

    def step_output(self, step: int, with_mt: bool = True):
        n = C.c_int64(0)
        rc = lib.ft_step_output(self.h, step, 0, None, None, None, None, C.byref(n))
        if rc not in (OK, ESIZE):
            self._chk(rc)
        _, par = self.step_inputs(step)  # params {kind, KA, KB, KC, nseg, nblk}
        so = np.empty(int(par[4]) + 1, np.int64)
        m = np.empty(n.value, np.int64) if with_mt else None
        t = np.empty(n.value, np.int64) if with_mt else None
        bp = np.empty(n.value, np.uint64)
        self._chk(lib.ft_step_output(self.h, step, n.value, _p(so, C.c_int64), _p(m, C.c_int64),
                                     _p(t, C.c_int64), _p(bp, C.c_uint64), C.byref(n)))
        return so, m, t, bp


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib.ft_nccl_unique_id(buf)
    if rc:
        raise FTError(rc, "ncclGetUniqueId")
    return buf.raw


def nccl_comm_init(world: int, rank: int, uid: bytes, device: int):
    c = C.c_void_p()
    rc = lib.ft_nccl_comm_init(world, rank, uid, device, C.byref(c))
    if rc:
        raise FTError(rc, "ncclCommInitRank")
    return c.value


def nccl_comm_destroy(comm):
    lib.ft_nccl_comm_destroy(C.c_void_p(comm))


def concat_costs(w):
    """(op_m, op_t, edge_m | None, edge_t) concatenated for ft_set_costs_all."""
    op_m = np.concatenate(w.op_m)
    op_t = np.concatenate(w.op_t)
    edge_t = np.concatenate(w.edge_t) if w.n_edges else np.zeros(0, np.int64)
    edge_m = None if w.edge_m is None else np.concatenate(w.edge_m)
    return op_m, op_t, edge_m, edge_t


def load(w, bulk: bool = True, costs=None, **kw) -> Graph:
    """Create a graph from a ``synth.graphs.Workload`` and upload its costs
    (one ft_set_costs_all call, or per-operator/per-edge setters)."""
    g = Graph(w.n_cfgs, w.src, w.dst, **kw)
    if bulk:
        g.set_costs_all(*(costs if costs is not None else concat_costs(w)))
        return g
    for i in range(w.n_ops):
        g.set_op_costs(i, w.op_m[i], w.op_t[i])
    for e in range(w.n_edges):
        g.set_edge_costs(e, None if w.edge_m is None else w.edge_m[e], w.edge_t[e])
    return g


def run_ft(w, **kw):
    """FT_AUTO eliminations + LDP + final reduce; returns (graph, m, t)."""
    g = load(w, **kw)
    g.eliminate(AUTO)
    m, t = g.frontier()
    return g, m, t


# ---------------------------------------------------------------------------
# Edge-cost generation (csrc/ft_costgen.cu)
# ---------------------------------------------------------------------------
def comm_profile(prof) -> ft_comm_profile:
    """Pack {L, P, lat[7], bw[7][47]} into the C struct of include/ft.h."""
    p = ft_comm_profile()
    p.mesh_log2, p.P = int(prof["L"]), int(prof["P"])
    lat = np.asarray(prof["lat"], np.int64)
    bw = np.asarray(prof["bw"], np.int64)
    for c in range(CG_MAX_MESH + 1):
        p.latency_ns[c] = int(lat[c])
        for i in range(CG_MAX_P + 1):
            p.bw[c][i] = int(bw[c, i])
    return p


def _cg_check(rc: int, what: str):
    if rc != OK:
        raise FTError(rc, what)


def comm_time(prof, nbytes, group_log2) -> np.ndarray:
    """ft_comm_time: interpolated collective time in ns (R18), on the GPU."""
    b = np.ascontiguousarray(nbytes, np.int64).ravel()
    g = np.ascontiguousarray(np.broadcast_to(np.asarray(group_log2, np.int32), b.shape), np.int32)
    out = np.zeros(b.shape, np.int64)
    p = prof if isinstance(prof, ft_comm_profile) else comm_profile(prof)
    _cg_check(lib.ft_comm_time(C.byref(p), b.size, _p(b, C.c_int64), _p(g, C.c_int32),
                               _p(out, C.c_int64)), "ft_comm_time")
    return out


def split_states(dims, mesh_log2: int) -> np.ndarray:
    """ft_split_states: split states (R19) of a tensor, [S, ndims] int32 (host)."""
    d = np.ascontiguousarray(dims, np.int64)
    n = C.c_int64(0)
    rc = lib.ft_split_states(d.size, _p(d, C.c_int64), mesh_log2, 0, None, C.byref(n))
    if rc not in (OK, ESIZE):
        raise FTError(rc, "ft_split_states")
    out = np.zeros((n.value, d.size), np.int32)
    _cg_check(lib.ft_split_states(d.size, _p(d, C.c_int64), mesh_log2, n.value,
                                  _p(out, C.c_int32), C.byref(n)), "ft_split_states")
    return out


def reschedule_costs(prof, ndims, dims, elem_bytes, q_tensor, q_from, q_to) -> np.ndarray:
    """ft_reschedule_costs: t_x = d(from,to) + d(to,from) per query (Eq. 2, R19)."""
    nd = np.ascontiguousarray(ndims, np.int32)
    dm = np.ascontiguousarray(dims, np.int64).reshape(nd.size, CG_MAX_DIMS)
    eb = np.ascontiguousarray(elem_bytes, np.int64)
    qt, qf, qo = (np.ascontiguousarray(a, np.int32).ravel() for a in (q_tensor, q_from, q_to))
    if not qt.size == qf.size == qo.size:
        raise ValueError(f"query arrays differ in length: {qt.size}, {qf.size}, {qo.size}")
    if dm.shape[0] != eb.size:
        raise ValueError("dims / elem_bytes do not match ndims")
    out = np.zeros(qt.size, np.int64)
    p = prof if isinstance(prof, ft_comm_profile) else comm_profile(prof)
    _cg_check(lib.ft_reschedule_costs(C.byref(p), nd.size, _p(nd, C.c_int32), _p(dm, C.c_int64),
                                      _p(eb, C.c_int64), qt.size, _p(qt, C.c_int32),
                                      _p(qf, C.c_int32), _p(qo, C.c_int32), _p(out, C.c_int64)),
              "ft_reschedule_costs")
    return out


def reschedule_costs_dev(prof, ndims, dims, elem_bytes, n_q: int, q_tensor: int, q_from: int,
                         q_to: int, t_out: int, stream: int = 0) -> None:
    """ft_reschedule_costs_dev: queries / output are DEVICE pointers (ints,
    e.g. torch ``tensor.data_ptr()``), kernels on ``stream`` (cudaStream_t)."""
    nd = np.ascontiguousarray(ndims, np.int32)
    dm = np.ascontiguousarray(dims, np.int64).reshape(nd.size, CG_MAX_DIMS)
    eb = np.ascontiguousarray(elem_bytes, np.int64)
    p = prof if isinstance(prof, ft_comm_profile) else comm_profile(prof)
    _cg_check(lib.ft_reschedule_costs_dev(C.byref(p), nd.size, _p(nd, C.c_int32),
                                          _p(dm, C.c_int64), _p(eb, C.c_int64), int(n_q),
                                          C.c_void_p(q_tensor), C.c_void_p(q_from),
                                          C.c_void_p(q_to), C.c_void_p(t_out),
                                          C.c_void_p(stream)), "ft_reschedule_costs_dev")


def sync_costs(prof, ndims, dims, elem_bytes, q_tensor, q_state):
    """ft_sync_costs: (m_p, t_s) of a parameter tensor per split state (Eq. 1, R20)."""
    nd = np.ascontiguousarray(ndims, np.int32)
    dm = np.ascontiguousarray(dims, np.int64).reshape(nd.size, CG_MAX_DIMS)
    eb = np.ascontiguousarray(elem_bytes, np.int64)
    qt, qs = (np.ascontiguousarray(a, np.int32).ravel() for a in (q_tensor, q_state))
    if qt.size != qs.size:
        raise ValueError(f"query arrays differ in length: {qt.size}, {qs.size}")
    if dm.shape[0] != eb.size:
        raise ValueError("dims / elem_bytes do not match ndims")
    m = np.zeros(qt.size, np.int64)
    t = np.zeros(qt.size, np.int64)
    p = prof if isinstance(prof, ft_comm_profile) else comm_profile(prof)
    _cg_check(lib.ft_sync_costs(C.byref(p), nd.size, _p(nd, C.c_int32), _p(dm, C.c_int64),
                                _p(eb, C.c_int64), qt.size, _p(qt, C.c_int32), _p(qs, C.c_int32),
                                _p(m, C.c_int64), _p(t, C.c_int64)), "ft_sync_costs")
    return m, t


def costgen_profile(on: bool) -> None:
    """ft_costgen_profile: CUDA-event timing of ft_reschedule_costs_dev's kernels."""
    _cg_check(lib.ft_costgen_profile(1 if on else 0), "ft_costgen_profile")


def costgen_last_times():
    """ft_costgen_last_times -> (apsp_ms, gather_ms) of the last profiled device call."""
    a, g = C.c_float(0), C.c_float(0)
    _cg_check(lib.ft_costgen_last_times(C.byref(a), C.byref(g)), "ft_costgen_last_times")
    return a.value, g.value
