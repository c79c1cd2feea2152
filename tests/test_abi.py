"""The C ABI library builds, loads and exports every symbol include/lsgpu.h declares (CPU only)."""

import ctypes
import os
import re

import pytest

from paper_2601_05709_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lsgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char \*)\s*\**(lsg_\w+)\(", text, re.M)))


def test_library_present():
    assert os.path.exists(_lib.LIB_PATH), "build liblsgpu.so first (make -C paper_2601_05709_b200/csrc)"


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"


def test_host_only_entry_points():
    lib = _lib.load(require_device=False)
    assert lib.lsg_abi_version() == 2
    g = _lib.make_grid(2, (160, 80), (0.0, 0.0), (2.0, 1.0))
    assert lib.lsg_num_nodes(g) == 161 * 81
    assert lib.lsg_num_elements(g) == 2 * 160 * 80
    assert lib.lsg_partials_per_rhs(g) >= 1024
    g3 = _lib.make_grid(3, (4, 3, 2), (0.0, 0.0, 0.0), (2.0, 1.0, 1.0))
    assert lib.lsg_num_nodes(g3) == 5 * 4 * 3
    assert lib.lsg_num_elements(g3) == 6 * 24
    bad = _lib.make_grid(2, (0, 8), (0.0, 0.0), (1.0, 1.0))
    assert lib.lsg_num_nodes(bad) == -1
    assert b"cell counts" in lib.lsg_last_error()


def test_product_refuses_cpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeUnavailable):
        _lib.load()
