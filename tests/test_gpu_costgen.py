"""GPU parity of edge-cost generation against the oracle:
ft_comm_time (R18) and ft_reschedule_costs (P:860 + Eq. 2, R19)
through the C-ABI, bit-exact (int64 ns)."""
import numpy as np
import pytest

import oracle
from synth import comm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ft():
    import paper_2004_10856_b200 as ft
    return ft


def _bytes(seed, n, P):
    rng = np.random.default_rng(seed)
    b = rng.integers(0, 2 ** P + 1, n)
    b[:P + 1] = 2 ** np.arange(P + 1)                 # every profile point
    b[P + 1:2 * P + 1] = 2 ** np.arange(1, P + 1) - 1  # just below each point
    b[2 * P + 1] = 0
    b[2 * P + 2: 2 * P + 200] = rng.integers(0, 4096, 198)  # latency regime
    return b.astype(np.int64)


@pytest.mark.parametrize("seed,L,P,monotone", [(0, 5, 40, False), (1, 6, 46, False),
                                                (2, 3, 30, True), (3, 1, 12, False)])
def test_comm_time_parity(ft, seed, L, P, monotone):
    prof = comm.profile(seed, L=L, P=P, monotone=monotone)
    b = _bytes(seed, 200_000, P)
    g = np.random.default_rng(seed + 9).integers(0, L + 1, b.size).astype(np.int32)
    assert np.array_equal(ft.comm_time(prof, b, g), oracle.comm_time(prof, b, g))


def test_comm_time_errors(ft):
    prof = comm.profile(0, L=3, P=20)
    with pytest.raises(ft.FTError) as e:
        ft.comm_time(prof, [2 ** 20 + 1], 1)
    assert e.value.code == ft.EOVERFLOW
    with pytest.raises(ft.FTError) as e:
        ft.comm_time(prof, [5], 4)
    assert e.value.code == ft.EINVAL
    assert ft.comm_time(prof, np.zeros(0, np.int64), 1).size == 0


def _tensor_set(seed, n, L, max_ndims=4):
    nd, dims, eb = comm.tensors(seed, n, L, max_ndims)
    ns = [len(oracle.split_states(dims[x, :nd[x]], L)) for x in range(n)]
    return nd, dims, eb, ns


@pytest.mark.parametrize("seed,L,n_t,n_q", [(0, 2, 7, 5000), (1, 3, 40, 100_000),
                                            (2, 5, 60, 300_000), (3, 4, 300, 200_000)])
def test_reschedule_parity(ft, seed, L, n_t, n_q):
    prof = comm.profile(seed, L=L, P=40)
    nd, dims, eb, ns = _tensor_set(seed, n_t, L)
    qt, qf, qo = comm.queries(seed, ns, n_q)
    got = ft.reschedule_costs(prof, nd, dims, eb, qt, qf, qo)
    want = oracle.reschedule_costs(prof, nd, dims, eb, qt, qf, qo)
    assert np.array_equal(got, want)


def test_reschedule_all_pairs_largest_state_graph(ft):
    # D = 4, L = 5, dims divisible by 32: C(9, 4) = 126 states, every pair.
    prof = comm.profile(11, L=5, P=44)
    dims = np.array([[64, 96, 32, 128], [3, 5, 7, 1], [1024, 1, 1, 1]], np.int64)
    nd = np.array([4, 4, 1], np.int32)
    eb = np.array([2, 4, 4], np.int64)
    for x in range(3):
        S = len(oracle.split_states(dims[x, :nd[x]], 5))
        f, t = np.meshgrid(np.arange(S), np.arange(S), indexing="ij")
        qt = np.full(S * S, x, np.int32)
        got = ft.reschedule_costs(prof, nd, dims, eb, qt, f.ravel(), t.ravel())
        want = oracle.reschedule_costs(prof, nd, dims, eb, qt, f.ravel(), t.ravel())
        assert np.array_equal(got, want), x
        if x == 0:
            assert S == 126
        if x == 1:
            assert S == 1 and got.tolist() == [0]


def test_reschedule_mesh64(ft):
    prof = comm.profile(5, L=6, P=46)
    nd, dims, eb, ns = _tensor_set(5, 50, 6, max_ndims=3)
    qt, qf, qo = comm.queries(5, ns, 50_000)
    assert np.array_equal(ft.reschedule_costs(prof, nd, dims, eb, qt, qf, qo),
                          oracle.reschedule_costs(prof, nd, dims, eb, qt, qf, qo))


def test_reschedule_errors(ft):
    prof = comm.profile(0, L=6, P=46)
    nd = np.array([4], np.int32)
    dims = np.array([[64, 64, 64, 64]], np.int64)    # C(10, 4) = 210 > 160 states
    eb = np.array([2], np.int64)
    z = np.zeros(1, np.int32)
    with pytest.raises(ft.FTError) as e:
        ft.reschedule_costs(prof, nd, dims, eb, z, z, z)
    assert e.value.code == ft.ESIZE
    with pytest.raises(ft.FTError) as e:
        ft.reschedule_costs(prof, np.array([1], np.int32), np.array([[4, 1, 1, 1]]), eb,
                            z, np.array([3], np.int32), z)   # state 3 of 3
    assert e.value.code == ft.EINVAL
    p20 = comm.profile(0, L=2, P=20)
    with pytest.raises(ft.FTError) as e:
        ft.reschedule_costs(p20, np.array([1], np.int32), np.array([[2 ** 20, 1, 1, 1]]), eb,
                            z, z, z)                         # 2^21 bytes > 2^P
    assert e.value.code == ft.EOVERFLOW
    out = ft.reschedule_costs(prof, nd[:0], dims[:0], eb[:0], z[:0], z[:0], z[:0])
    assert out.size == 0


def test_generated_edge_costs_drive_ft(ft):
    """Generated t_x tables (Eq. 2, m = 0) feed a search: a chain whose edge
    costs come from ft_reschedule_costs gives the oracle's frontier."""
    from synth import graphs as G
    w = G.c2(seed=0)
    L = 3
    prof = comm.profile(3, L=L, P=44)
    rng = np.random.default_rng(3)
    n_e = len(w.src)
    nd = np.full(n_e, 2, np.int32)
    dims = np.ones((n_e, 4), np.int64)
    dims[:, 0], dims[:, 1] = 256, 1024
    eb = np.full(n_e, 2, np.int64)
    S = len(oracle.split_states([256, 1024], L))
    # each op config picks an output split and a required input split
    out_state = [rng.integers(0, S, k) for k in w.n_cfgs]
    in_state = [rng.integers(0, S, k) for k in w.n_cfgs]
    qt, qf, qo = [], [], []
    for e, (s, d) in enumerate(zip(w.src, w.dst)):
        f, t = np.meshgrid(out_state[s], in_state[d], indexing="ij")
        qt.append(np.full(f.size, e)); qf.append(f.ravel()); qo.append(t.ravel())
    qt, qf, qo = (np.concatenate(a).astype(np.int32) for a in (qt, qf, qo))
    tx = ft.reschedule_costs(prof, nd, dims, eb, qt, qf, qo)
    assert np.array_equal(tx, oracle.reschedule_costs(prof, nd, dims, eb, qt, qf, qo))
    off = 0
    edge_t = []
    for s, d in zip(w.src, w.dst):
        n = int(w.n_cfgs[s]) * int(w.n_cfgs[d])
        edge_t.append(tx[off:off + n].copy()); off += n
    import dataclasses
    w2 = dataclasses.replace(w, edge_t=edge_t, edge_m=None).check()
    g, m, t = ft.run_ft(w2)
    og, om, ot = oracle.run_ft(w2, threads=4)
    assert np.array_equal(m, om) and np.array_equal(t, ot)


def test_reschedule_dev_pointers(ft):
    """ft_reschedule_costs_dev: device queries/output on a torch stream."""
    import torch
    prof = comm.profile(6, L=4, P=40)
    nd, dims, eb, ns = _tensor_set(6, 100, 4)
    qt, qf, qo = comm.queries(6, ns, 123_457)
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(a).to(dev) for a in (qt, qf, qo)]
    out = torch.full((qt.size,), -1, dtype=torch.int64, device=dev)
    s = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    ft.reschedule_costs_dev(prof, nd, dims, eb, qt.size, d[0].data_ptr(), d[1].data_ptr(),
                            d[2].data_ptr(), out.data_ptr(), s.cuda_stream)
    want = oracle.reschedule_costs(prof, nd, dims, eb, qt, qf, qo)
    assert np.array_equal(out.cpu().numpy(), want)
    bad = d[1].clone()
    bad[777] = 10_000                                   # out-of-range state, caught on device
    with pytest.raises(ft.FTError) as e:
        ft.reschedule_costs_dev(prof, nd, dims, eb, qt.size, d[0].data_ptr(), bad.data_ptr(),
                                d[2].data_ptr(), out.data_ptr(), s.cuda_stream)
    assert e.value.code == ft.EINVAL


@pytest.mark.parametrize("seed,L", [(0, 3), (1, 5), (2, 6)])
def test_sync_costs_parity(ft, seed, L):
    """ft_sync_costs (Eq. 1 m_p / t_s, R20) bit-exact vs the oracle."""
    prof = comm.profile(seed, L=L, P=44)
    nd, dims, eb, ns = _tensor_set(seed, 80, L, max_ndims=3)
    qt, qs, _ = comm.queries(seed, ns, 60_000)
    m, t = ft.sync_costs(prof, nd, dims, eb, qt, qs)
    om, ot = oracle.sync_costs(prof, nd, dims, eb, qt, qs)
    assert np.array_equal(m, om) and np.array_equal(t, ot)
    with pytest.raises(ft.FTError) as e:
        ft.sync_costs(prof, nd, dims, eb, qt[:1], np.array([10_000], np.int32))
    assert e.value.code == ft.EINVAL


def test_costgen_profile_times(ft):
    """ft_costgen_profile / ft_costgen_last_times report both kernels' times."""
    import torch
    prof = comm.profile(7, L=3, P=40)
    nd, dims, eb, ns = _tensor_set(7, 30, 3)
    qt, qf, qo = comm.queries(7, ns, 200_000)
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(a).to(dev) for a in (qt, qf, qo)]
    out = torch.empty(qt.size, dtype=torch.int64, device=dev)
    ft.costgen_profile(True)
    try:
        ft.reschedule_costs_dev(prof, nd, dims, eb, qt.size, d[0].data_ptr(), d[1].data_ptr(),
                                d[2].data_ptr(), out.data_ptr(), 0)
        a, g = ft.costgen_last_times()
    finally:
        ft.costgen_profile(False)
    assert a > 0 and g > 0
    assert np.array_equal(out.cpu().numpy(), oracle.reschedule_costs(prof, nd, dims, eb, qt, qf, qo))


@pytest.mark.parametrize("L", [5, 6])
def test_costgen_fullsize_bench_workload(ft, L):
    """Full-size parity at the bench configuration (tools/bench_costgen.py,
    CG5: 9.52 M queries, the launch configuration it times), host-buffer and
    device-pointer entries, every query against the oracle."""
    import os
    import sys
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    import bench_costgen as B
    w, nd, dims, eb, rng = B.workload(0, L)
    ns = [len(ft.split_states(dims[x, :nd[x]], L)) for x in range(len(nd))]
    qt, qf, qo = B.queries(w, ns, rng)
    prof = comm.profile(0, L=L, P=40)
    want = oracle.reschedule_costs(prof, nd, dims, eb, qt, qf, qo)
    assert np.array_equal(ft.reschedule_costs(prof, nd, dims, eb, qt, qf, qo), want)
    dev = torch.device("cuda:0")
    d = [torch.from_numpy(a).to(dev) for a in (qt, qf, qo)]
    out = torch.empty(qt.size, dtype=torch.int64, device=dev)
    ft.reschedule_costs_dev(prof, nd, dims, eb, qt.size, d[0].data_ptr(), d[1].data_ptr(),
                            d[2].data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(out.cpu().numpy(), want)
