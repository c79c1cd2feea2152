"""The reference-side ctypes binding documented in INTEGRATION.md section 2, executed
verbatim: struct mirrors against the library's own sizeof exports, and its
csr_free_apply against the oracle's assembled, Dirichlet-eliminated CSR K @ u
(reference fem.py:141-150,274-291,397-411) on a reference-shaped RectMesh."""

import os
import re
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def documented_stub():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("### The binding a reference maintainer would add"):]
    return re.search(r"```python\n(.*?)```", sec, re.S).group(1)


def test_documented_stub_runs_and_matches_csr(monkeypatch):
    pytest.importorskip("torch")
    from paper_2601_05709_b200 import _lib
    from oracle import fem as ofem, model as omodel
    from oracle.grid import Grid

    _lib.load()  # the product's own binding also asserts the sizes
    monkeypatch.setenv("LSGPU_LIB", _lib.LIB_PATH)
    ns = {}
    exec(compile(documented_stub(), "INTEGRATION.md", "exec"), ns)
    nx, ny = 40, 20
    rules = [(1, lambda p: p[:, 0] < 1e-12)]
    grid = Grid((0.0, 0.0), (2.0, 1.0), (nx, ny), rules)
    space = ofem.Space(grid, 2)
    clamp = ofem.clamp_dofs(space, grid.facets_with_tag(1))
    phi = np.random.default_rng(3).standard_normal(grid.num_vertices) - 0.2
    lame = (0.3 / 0.91, 1.0 / 2.6)
    model = omodel.Compliance(grid, lame, 1e-3, clamp, [], 1.0)
    K, _ = ofem.dirichlet_eliminate(model.matrix(phi), np.zeros(space.dof_count), clamp)
    mesh = SimpleNamespace(bounds=(0.0, 0.0, 2.0, 1.0), nx=nx, ny=ny, num_vertices=grid.num_vertices)
    u = np.random.default_rng(4).standard_normal(space.dof_count)
    y = ns["csr_free_apply"](mesh, phi, u, lame, 1e-3, clamp)
    assert rel_l2(y, K @ u) <= 1e-10


def test_sizeof_exports_match_product_mirrors():
    import ctypes
    from paper_2601_05709_b200 import _lib
    lib = _lib.load()
    assert lib.lsg_sizeof_op() == ctypes.sizeof(_lib.Op) == 160
    assert lib.lsg_sizeof_grid() == ctypes.sizeof(_lib.Grid)
    assert lib.lsg_sizeof_pcg_ws() == ctypes.sizeof(_lib.PcgWs)
