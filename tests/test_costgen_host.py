"""Host-side logic of libft's edge-cost generation (no GPU needed): the split
state enumeration (R19) against the oracle's, and the argument checks that
return before any device work (include/ft.h)."""
import numpy as np
import pytest

import oracle
from synth import comm


@pytest.fixture(scope="module")
def ft():
    import paper_2004_10856_b200 as ft
    return ft


def test_split_states_match_oracle(ft):
    for L in range(1, 7):
        nd, dims, _ = comm.tensors(L, 200, L)
        for x in range(200):
            d = dims[x, :nd[x]]
            assert np.array_equal(ft.split_states(d, L), oracle.split_states(d, L)), (L, d)


def test_split_states_errors(ft):
    with pytest.raises(ft.FTError):
        ft.split_states([4, 4, 4, 4, 4], 2)     # more than FT_CG_MAX_DIMS dims
    with pytest.raises(ft.FTError):
        ft.split_states([4], 7)                 # mesh above 2^6
    with pytest.raises(ft.FTError):
        ft.split_states([0], 2)


def test_reschedule_host_errors(ft):
    prof = comm.profile(0, L=6, P=46)
    z = np.zeros(1, np.int32)
    eb = np.array([2], np.int64)
    with pytest.raises(ft.FTError) as e:        # C(10, 4) = 210 > 160 states
        ft.reschedule_costs(prof, np.array([4], np.int32), np.array([[64] * 4]), eb, z, z, z)
    assert e.value.code == ft.ESIZE
    p20 = comm.profile(0, L=2, P=20)
    with pytest.raises(ft.FTError) as e:        # 2^21 bytes > 2^P
        ft.reschedule_costs(p20, np.array([1], np.int32), np.array([[2 ** 20, 1, 1, 1]]), eb,
                            z, z, z)
    assert e.value.code == ft.EOVERFLOW
    bad = comm.profile(0, L=2, P=20)
    bad["bw"][1, 3] = 0                          # bandwidth must be > 0
    with pytest.raises(ft.FTError) as e:
        ft.reschedule_costs(bad, np.array([1], np.int32), np.array([[4, 1, 1, 1]]), eb, z, z, z)
    assert e.value.code == ft.EINVAL
    with pytest.raises(ft.FTError) as e:
        ft.comm_time(bad, [5], 1)
    assert e.value.code == ft.EINVAL
    with pytest.raises(ft.FTError) as e:
        ft.comm_time(p20, [2 ** 20 + 1], 1)
    assert e.value.code == ft.EOVERFLOW


def test_query_length_checked_in_binding(ft):
    """Mismatched query arrays are rejected before any pointer crosses the ABI."""
    prof = comm.profile(0, L=2, P=20)
    nd, dims, eb = np.array([1], np.int32), np.array([[4, 1, 1, 1]]), np.array([2], np.int64)
    z = np.zeros(3, np.int32)
    with pytest.raises(ValueError):
        ft.reschedule_costs(prof, nd, dims, eb, z, z[:2], z)
    with pytest.raises(ValueError):
        ft.sync_costs(prof, nd, dims, eb, z, z[:1])
    with pytest.raises(ValueError):
        ft.sync_costs(prof, nd, dims, np.array([2, 2], np.int64), z, z)
