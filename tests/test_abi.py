"""CPU checks of the C-ABI boundary: the in-tree library loads without a
GPU and exports every function include/card_b200.h declares."""

import ctypes
import os
import re

from conftest import ROOT


def declared_functions():
    with open(os.path.join(ROOT, "include", "card_b200.h")) as fh:
        src = fh.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(card_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2508_04462_b200._lib import LIB_PATH, SIGNATURES, raw

    assert os.path.exists(LIB_PATH), "run __graft_entry__.build() first"
    handle = raw()
    decl = declared_functions()
    assert decl, "no declarations parsed"
    for name in decl:
        assert hasattr(handle, name), f"{name} declared but not exported"
        assert name in SIGNATURES, f"{name} has no ctypes signature"
    assert set(SIGNATURES) <= set(decl)
    assert handle.card_abi_version() == 1
    assert handle.card_strerror(-4) == b"frontier full"


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        return
    import pytest

    import paper_2508_04462_b200 as card

    with pytest.raises(card.DeviceError):
        card.TreeCache(0, card.CacheConfig(2, 2, 2))
