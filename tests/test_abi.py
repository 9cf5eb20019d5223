"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/btree.h declares, and validates arguments before any
device work (BT_ERR_ARG paths)."""
import ctypes as C
import os
import re

import pytest

import paper_1910_02639_b200 as P
from paper_1910_02639_b200 import btree

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "btree.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bt_[a-z_]+)\s*\(", src)))


def test_header_declares_the_abi():
    names = declared()
    for must in ("bt_build", "bt_find_neighbors", "bt_free"):
        assert must in names
    assert sorted(btree.EXPORTS) == names


def test_library_exports_every_declared_symbol():
    L = P.lib()
    for name in declared():
        assert hasattr(L, name), name
        assert C.cast(getattr(L, name), C.c_void_p).value


def test_argument_errors_without_device():
    L = P.lib()
    assert not L.bt_build(None, -1, 64, 0.5)
    assert L.bt_last_status() == btree.BT_ERR_ARG
    assert b"n" in L.bt_last_error()
    assert not L.bt_build(None, 10, 64, 0.5)          # pos NULL with n > 0
    assert L.bt_last_status() == btree.BT_ERR_ARG
    assert not L.bt_build_ex(None, 0, 0, 0.5, 0.5, 64)  # s < 1
    assert not L.bt_build_ex(None, 0, 8, 1.5, 0.5, 64)  # beta > 1
    assert not L.bt_build_ex(None, 0, 8, 0.5, -0.1, 64)  # alpha < 0
    assert L.bt_find_neighbors(None, None, 1, None, None, None) == btree.BT_ERR_ARG
    assert L.bt_fill_neighbors(None, None, None, None, 0) == btree.BT_ERR_ARG
    assert L.bt_find_neighbors_sym(None, None, 1, None, None, None) == btree.BT_ERR_ARG
    assert L.bt_fill_neighbors_sym(None, None, None, None, 0) == btree.BT_ERR_ARG
    assert L.bt_density(None, None, None, None) == btree.BT_ERR_ARG
    assert L.bt_set_partition(None, 0, 1) == btree.BT_ERR_ARG
    assert L.bt_set_tree_order(None, 1) == btree.BT_ERR_ARG
    assert L.bt_reorder(None, None, 1, None) == btree.BT_ERR_ARG
    for bad_policy in (-1, 4):  # BT_POLICY_BTREE .. BT_POLICY_QUADTREE
        assert not L.bt_build_policy(None, 0, 8, 0.5, 0.5, 64, bad_policy)
        assert L.bt_last_status() == btree.BT_ERR_ARG
    assert L.bt_tree_stats(None, None) == btree.BT_ERR_ARG
    assert L.bt_search_host(None, None, -1, 64, 0.5, None, None, None, 0) == btree.BT_ERR_ARG
    L.bt_free(None)  # NULL-safe
    assert L.bt_set_stream(None) == btree.BT_OK
    assert L.bt_profile_enable(0) == btree.BT_OK


def test_binding_rejects_cpu_tensors():
    torch = pytest.importorskip("torch")
    with pytest.raises(TypeError):
        P.build(torch.zeros((4, 3), dtype=torch.float64))
