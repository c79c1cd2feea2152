"""Large grids (edge case: sizes far beyond the BASELINE configs): a 67M-dof 2D
and a 43M-dof 3D (k = 2) operator stay symmetric to round-off and the batched
PCG converges, with int64 indexing throughout.  Needs a B200 (~15 GB)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

lsg = pytest.importorskip("paper_2601_05709_b200")
from paper_2601_05709_b200 import (DirichletSet, ElasticityOperator, FunctionSpace,  # noqa: E402
                                   build_box_mesh, build_rect_mesh)
from paper_2601_05709_b200.fem import solve_batched  # noqa: E402


@pytest.mark.parametrize("dim", [2, 3])
def test_large_grid_symmetry_and_solve(dim):
    clamp = [(1, lambda p: p[:, 0] < 1e-12)]
    if dim == 2:
        mesh, lame, k = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 8192, 4096, clamp), (0.33, 0.38), 1
    else:
        mesh, lame, k = build_box_mesh((0, 0, 0, 2, 1, 1), (384, 192, 192), clamp), (0.58, 0.38), 2
    space = FunctionSpace(mesh, dim)
    g = torch.Generator(device="cuda").manual_seed(0)
    phi = torch.randn(mesh.num_vertices, dtype=torch.float64, device="cuda", generator=g)
    op = ElasticityOperator(space, phi, lame, 1e-3, DirichletSet.on_tags(space, 1))
    u = torch.randn((k, space.dof_count), dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn((k, space.dof_count), dtype=torch.float64, device="cuda", generator=g)
    Ku, Kv = op.apply(u), op.apply(v)
    vku, ukv = float((v * Ku).sum()), float((u * Kv).sum())
    assert abs(vku - ukv) <= 1e-13 * abs(vku)
    x, it = solve_batched(op, Ku, rtol=1e-6, maxiter=5000)
    for r in range(k):
        res = float(torch.linalg.vector_norm(Ku[r] - op.apply(x[r])))
        assert res <= 2e-6 * float(torch.linalg.vector_norm(Ku[r]))
        assert int(it[r]) > 10
