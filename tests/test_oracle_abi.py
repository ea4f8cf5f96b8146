"""Oracle ABI error behaviour (mirrors include/ft.h conventions)."""
import numpy as np
import pytest

import oracle
from synth import graphs as G


def test_errors():
    with pytest.raises(oracle.OracleError):
        oracle.Graph([2, 2], [0], [0])  # src == dst
    with pytest.raises(oracle.OracleError):
        oracle.Graph([2, 2], [0, 1], [1, 0])  # cycle
    g = oracle.Graph([2, 2], [0], [1])
    with pytest.raises(oracle.OracleError) as e:
        g.eliminate()
    assert e.value.code == oracle.ESTATE  # missing costs
    g.set_op_costs(0, [1, 2], [3, 4])
    with pytest.raises(oracle.OracleError) as e:
        g.set_op_costs(1, [-1, 2], [3, 4])
    assert e.value.code == oracle.EINVAL
    with pytest.raises(oracle.OracleError) as e:
        g.set_op_costs(1, [1 << 40, 2], [3, 4])
    assert e.value.code == oracle.EOVERFLOW
    g.set_op_costs(1, [1, 2], [3, 4])
    g.set_edge_costs(0, None, [0, 1, 1, 0])
    with pytest.raises(oracle.OracleError) as e:
        g.eliminate(oracle.NODE, 0)
    assert e.value.code == oracle.EPRECOND
    with pytest.raises(oracle.OracleError) as e:
        g.eliminate(oracle.EDGE, 0)
    assert e.value.code == oracle.EPRECOND
    m, t = g.frontier()
    assert len(m) >= 1
    with pytest.raises(oracle.OracleError) as e:
        g.set_op_costs(0, [1, 2], [3, 4])
    assert e.value.code == oracle.ESTATE


def test_not_linear():
    # the bridge DAG (non-series-parallel, every op of degree >= 2) with K = 65:
    # no node, edge, K=1-fold or leaf branch elimination applies, and a
    # composite configuration space would exceed 4096 (R21) -> not linear
    w = G.random_graph(4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], 65, 0)
    g = oracle.load(w)
    g.eliminate()
    with pytest.raises(oracle.OracleError) as e:
        g.frontier()
    assert e.value.code == oracle.EPRECOND
