"""libft's C-ABI contract on the GPU (include/ft.h conventions):
every error class, the two-call size pattern, the strong guarantee (a failed
call leaves the graph unchanged), handle poisoning, and the device-memory
hooks (ft_options.alloc / .free).  Calls go through the ctypes binding or
straight to ``ft.lib``."""
import ctypes as C

import numpy as np
import pytest

import oracle
from synth import graphs as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ft():
    import paper_2004_10856_b200 as ft
    return ft


def code(fn, *a, **kw):
    """Return the FTError code raised by fn (0 if it succeeds)."""
    import paper_2004_10856_b200 as ft
    try:
        fn(*a, **kw)
    except ft.FTError as e:
        return e.code
    return 0


def reference(w):
    og = oracle.load(w, 4)
    og.eliminate()
    return og.frontier()


def same_frontier(g, w):
    m, t = g.frontier()
    om, ot = reference(w)
    return np.array_equal(m, om) and np.array_equal(t, ot)


def test_create_errors(ft):
    assert code(ft.Graph, [2, 2], [0], [0]) == ft.EINVAL          # src == dst
    assert code(ft.Graph, [2, 2], [0, 1], [1, 0]) == ft.EINVAL    # cycle
    assert code(ft.Graph, [2, 0], [0], [1]) == ft.EINVAL          # K < 1
    assert code(ft.Graph, [2, 4097], [0], [1]) == ft.EINVAL       # K > 4096
    assert code(ft.Graph, [2, 2], [0], [5]) == ft.EINVAL          # bad endpoint
    n = 1 << 19
    src = np.arange(n, dtype=np.int32)
    assert code(ft.Graph, np.ones(n + 1, np.int32), src, src + 1) == ft.EOVERFLOW  # n_ops + n_edges >= 2^20
    a, f = ft.torch_allocator()
    assert code(ft.Graph, [2, 2], [0], [1], alloc=(a, None)) == ft.EINVAL  # hooks come in pairs


def test_cost_errors_and_strong_guarantee(ft):
    w = G.c1(3)
    g = ft.Graph(w.n_cfgs, w.src, w.dst)
    assert code(g.eliminate) == ft.ESTATE                          # costs missing
    assert code(g.frontier) == ft.ESTATE
    for i in range(w.n_ops):
        g.set_op_costs(i, w.op_m[i], w.op_t[i])
    bad = w.op_m[0].copy()
    bad[1] = -1
    assert code(g.set_op_costs, 0, bad, w.op_t[0]) == ft.EINVAL     # negative
    bad[1] = 1 << 40
    assert code(g.set_op_costs, 0, bad, w.op_t[0]) == ft.EOVERFLOW  # R10
    assert code(g.set_op_costs, 9, w.op_m[0], w.op_t[0]) == ft.EINVAL
    assert code(g.set_edge_costs, 0, None, -w.edge_t[0] - 1) == ft.EINVAL
    assert code(g.set_edge_costs, 7, None, w.edge_t[0]) == ft.EINVAL
    for e in range(w.n_edges):
        g.set_edge_costs(e, None, w.edge_t[e])
    assert code(g.set_costs_all, *ft.concat_costs(w)) == ft.ESTATE  # only one cost setter
    # preconditions: o_0 is marked / has no in-edge; no parallel edge
    assert code(g.eliminate, ft.NODE, 0) == ft.EPRECOND
    assert code(g.eliminate, ft.EDGE, 0) == ft.EPRECOND
    assert code(g.eliminate, ft.NODE, 17) == ft.EINVAL
    assert code(g.eliminate, 99) == ft.EINVAL                       # bad kind
    assert code(g.strategy, 0) == ft.ESTATE                         # before ft_frontier
    assert code(g.mini_time, 10) == ft.ESTATE
    # none of the failures above changed the graph
    g.eliminate()
    assert same_frontier(g, w)
    assert code(g.set_op_costs, 0, w.op_m[0], w.op_t[0]) == ft.ESTATE  # after elimination
    assert code(g.eliminate) == ft.ESTATE                           # frontier already computed
    assert code(g.frontier, "elim") == ft.ESTATE                    # one final frontier per graph
    assert code(g.strategy, 10 ** 6) == ft.EINVAL
    assert code(g.strategy, -1) == ft.EINVAL
    assert same_frontier(g, w)


def test_bulk_cost_errors_leave_graph_unset(ft):
    w = G.c3()
    g = ft.Graph(w.n_cfgs, w.src, w.dst)
    op_m, op_t, em, et = ft.concat_costs(w)
    bad = op_t.copy()
    bad[5] = -3
    assert code(g.set_costs_all, op_m, bad, em, et) == ft.EINVAL    # validated on the device
    bad[5] = (1 << 40) + 1
    assert code(g.set_costs_all, op_m, bad, em, et) == ft.EOVERFLOW
    assert code(g.eliminate) == ft.ESTATE                           # still no costs
    g.set_costs_all(op_m, op_t, em, et)                             # then the real ones
    g.eliminate()
    assert same_frontier(g, w)


def test_not_linear_is_eprecond_and_recoverable_state(ft):
    # the bridge DAG at K = 65: no exact elimination makes it a chain (a
    # composite configuration space would exceed 4096, R21)
    w = G.random_graph(4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], 65, 0)
    g = ft.load(w)
    g.eliminate()
    assert code(g.frontier) == ft.EPRECOND
    assert code(g.frontier) == ft.EPRECOND                          # not poisoned
    assert code(g.frontier, "elim") == ft.EPRECOND


def test_two_call_size_pattern(ft):
    w = G.c2()
    g = ft.load(w)
    g.eliminate()
    n = C.c_int64(-1)
    assert ft.lib.ft_frontier(g.h, 0, None, None, C.byref(n)) == ft.ESIZE
    need = n.value
    assert need > 1
    m = np.zeros(need - 1, np.int64)
    t = np.zeros(need - 1, np.int64)
    P = C.POINTER(C.c_int64)
    assert ft.lib.ft_frontier(g.h, need - 1, m.ctypes.data_as(P), t.ctypes.data_as(P), C.byref(n)) == ft.ESIZE
    assert n.value == need and not m.any()                          # nothing written
    m = np.zeros(need, np.int64)
    t = np.zeros(need, np.int64)
    assert ft.lib.ft_frontier(g.h, need, m.ctypes.data_as(P), t.ctypes.data_as(P), C.byref(n)) == ft.OK
    om, ot = reference(w)
    assert np.array_equal(m, om) and np.array_equal(t, ot)
    k = C.c_int64(-1)
    assert ft.lib.ft_get_stats(g.h, None, 0, C.byref(k)) in (ft.OK, ft.ESIZE)
    assert k.value == len(g.stats())
    buf = (ft.ft_step_stats * 1)()
    assert ft.lib.ft_get_stats(g.h, buf, 1, C.byref(k)) == ft.ESIZE
    assert ft.lib.ft_step_output(g.h, 0, 0, None, None, None, None, C.byref(k)) == ft.ESIZE
    assert ft.lib.ft_step_output(g.h, 10 ** 6, 0, None, None, None, None, C.byref(k)) == ft.EINVAL
    # consumed step m/t without keep_all
    so = np.zeros(1 << 12, np.int64)
    mm = np.zeros(1 << 20, np.int64)
    assert ft.lib.ft_step_output(g.h, 0, len(mm), so.ctypes.data_as(P), mm.ctypes.data_as(P), None, None,
                                 C.byref(k)) == ft.ESTATE


def test_torch_allocator_hook(ft):
    """Every device buffer through torch's caching allocator: same results,
    and the memory shows up in torch's accounting while the graph lives."""
    import torch
    w = G.c5(n_ops=300, K=32, B=8, Lmin=3, Lmax=8)
    a = ft.load(w)
    a.eliminate()
    am, at = a.frontier()
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    b = ft.load(w, torch_alloc=True, keep_all=True)
    b.eliminate()
    bm, bt = b.frontier()
    assert torch.cuda.memory_allocated() > before
    assert np.array_equal(am, bm) and np.array_equal(at, bt)
    for i in np.linspace(0, len(am) - 1, 8).astype(int):
        assert np.array_equal(a.strategy(int(i)), b.strategy(int(i)))
    for s in range(0, len(b.stats()), 17):
        for x, y in zip(a.step_output(s, with_mt=False), b.step_output(s, with_mt=False)):
            assert x is None or np.array_equal(x, y)
    b.close()
    a.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == before  # scratch and arenas handed back


def test_allocator_hook_oom_poisons(ft):
    """A hook that runs out of memory: FT_ENOMEM, then the handle is poisoned
    (every later call returns the same code); other handles are unaffected."""
    import torch
    calls = {"n": 0, "live": {}}
    budget = 6

    @ft.ALLOC_FN
    def alloc(nbytes, stream, ctx):
        calls["n"] += 1
        if calls["n"] > budget:
            return None
        p = torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(),
                                               torch.cuda.current_stream())
        calls["live"][p] = nbytes
        return p

    @ft.FREE_FN
    def free(p, stream, ctx):
        calls["live"].pop(p, None)
        torch.cuda.caching_allocator_delete(p)

    hooks = (C.cast(alloc, C.c_void_p).value, C.cast(free, C.c_void_p).value)
    w = G.c3()
    g = ft.load(w, alloc=hooks)
    rc = code(g.eliminate)
    assert rc == ft.ENOMEM
    assert code(g.frontier) == ft.ENOMEM
    assert code(g.eliminate) == ft.ENOMEM
    g.close()
    assert calls["live"] == {}                                      # everything handed back
    h = ft.load(w)                                                  # independent handle
    h.eliminate()
    assert same_frontier(h, w)
