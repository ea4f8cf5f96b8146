"""The C-ABI library loads on a CPU-only box and exports every function that
include/ft.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "ft.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ft_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ["ft_graph_create", "ft_set_op_costs", "ft_set_edge_costs", "ft_eliminate",
              "ft_frontier", "ft_strategy", "ft_graph_destroy", "ft_last_error", "ft_get_stats"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2004_10856_b200 as ft
    lib = ctypes.CDLL(ft.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert missing == []
    assert set(ft.SYMBOLS) == set(declared())
    assert ft.lib.ft_version().startswith(b"ft-b200")


def test_no_cpu_fallback():
    """Without a usable device the product path fails loudly (FT_ECUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2004_10856_b200 as ft
    with pytest.raises(ft.FTError) as e:
        ft.Graph([2, 2], [0], [1])
    assert e.value.code == ft.ECUDA


def test_host_only_entry_points():
    import numpy as np
    import paper_2004_10856_b200 as ft
    b = ft.shard_plan(np.array([3, 1, 4, 1, 5, 9, 2, 6]), 3)
    assert b[0] == 0 and b[-1] == 8
    with pytest.raises(ft.FTError):
        ft.shard_plan(np.array([1, -1]), 2)


def test_allocator_hooks_checked_before_device_use():
    """ft_options.alloc / .free come in pairs (FT_EINVAL), checked on the host."""
    import paper_2004_10856_b200 as ft
    dummy = ft.ALLOC_FN(lambda n, s, c: None)
    with pytest.raises(ft.FTError) as e:
        ft.Graph([2, 2], [0], [1], alloc=(ctypes.cast(dummy, ctypes.c_void_p).value, None))
    assert e.value.code == ft.EINVAL
    assert ctypes.sizeof(ft.ft_options) == 88  # include/ft.h layout (x86-64)


def test_torch_alloc_shim_exports():
    import paper_2004_10856_b200 as ft
    lib = ctypes.CDLL(ft.TORCH_ALLOC_PATH)
    assert hasattr(lib, "ft_torch_alloc") and hasattr(lib, "ft_torch_free")
