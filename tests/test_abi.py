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
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|void|const char \*)\s*\**(lsg_\w+)\(",
                                 text, re.M)))


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
    assert lib.lsg_abi_version() == 3
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


def _op(kind, dim=2, words=1):
    n = (8, 4) if dim == 2 else (4, 3, 2)
    lo, hi = (0.0,) * dim, (2.0, 1.0, 1.0)[:dim]
    op = _lib.Op()
    op.kind = kind
    op.grid = _lib.make_grid(dim, n, lo, hi)
    op.words = words or None  # never dereferenced: validation fails first
    for i in range(4):
        op.p[i] = 1.0
    return op


def test_argument_errors_are_reported_before_any_device_work():
    """The C ABI validates its arguments on the host and reports LSG_ERR_ARG with a
    message (ConfigError on the Python side), without touching the device."""
    lib = _lib.load(require_device=False)
    null = ctypes.c_void_p(None)
    cases = [
        (lambda: lib.lsg_apply(None, 1, null, null, null), b"null operator"),
        (lambda: lib.lsg_apply(_op(99), 1, null, null, null), b"unknown operator kind"),
        (lambda: lib.lsg_apply(_op(_lib.LSG_OP_ELASTICITY, words=0), 1, null, null, null),
         b"words missing"),
        (lambda: lib.lsg_apply(_op(_lib.LSG_OP_LAPLACE, dim=3), 1, null, null, null), b"2D only"),
        (lambda: lib.lsg_heat_shape(_op(_lib.LSG_OP_ELASTICITY), 1, null, null, null, null, 1.0,
                                    null, null, null, null, null, null), b"scalar diffusion"),
        (lambda: lib.lsg_shape_rhs(_op(_lib.LSG_OP_ELASTICITY), 1, null, 0.0, null, null, null,
                                   null, null, null, null), b"volume"),
        (lambda: lib.lsg_inverse_misfit(_lib.make_grid(3, (2, 2, 2), (0, 0, 0), (1, 1, 1)), 1, null,
                                        null, null, null, null, 1.0, 1.0, null, null, null, null,
                                        null, null), b"2D only"),
    ]
    for fn, msg in cases:
        assert fn() == _lib.LSG_ERR_ARG
        assert msg in lib.lsg_last_error(), (msg, lib.lsg_last_error())
