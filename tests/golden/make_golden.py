"""Generate golden vectors from the reference implementation (lsopt 0.1.0).

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/reference_2d.npz``.  Every array is produced by the
reference's own public API (mesh.py, fem.py, levelset.py, models/, velocity.py,
ppl.py, driver.py) on small seeded inputs; the oracle and the CUDA path are
checked against these in ``tests/test_oracle.py`` and ``tests/test_gpu_parity.py``.
The reference tree is not available on the GPU box, so only these files travel.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from lsopt import driver as ldriver  # noqa: E402
from lsopt.fem import (DirichletSet, FemField, FunctionSpace, SparseSystem, apply_dirichlet,  # noqa: E402
                       elasticity_matrix, vector_load)
from lsopt.levelset import LevelSetField  # noqa: E402
from lsopt.mesh import build_rect_mesh, mesh_diameter  # noqa: E402
from lsopt.models import ComplianceModel, CompliancePlusModel, MaterialIndicator  # noqa: E402
from lsopt.models.base import solve_problem  # noqa: E402
from lsopt.ppl import combine_derivatives, lagrangian_value, ppl_init, ppl_update  # noqa: E402
from lsopt.velocity import BilinearSpec, VelocitySolver  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_2d.npz")

LAME = (0.3 / 0.91, 1.0 / 2.6)  # plane stress, E = 1, nu = 0.3
ERSATZ = 1e-3


def cantilever(nx, ny):
    rules = [(1, lambda p: p[:, 0] < 1e-12),
             (2, lambda p: (p[:, 0] > 2.0 - 1e-12) & (p[:, 1] >= 0.45) & (p[:, 1] <= 0.55))]
    return build_rect_mesh((0.0, 0.0, 2.0, 1.0), nx, ny, rules)


def phi_fn(p):
    return -np.cos(6 * np.pi * p[:, 0]) * np.cos(4 * np.pi * p[:, 1]) - 0.4


def main():
    g = {}
    # -- mesh (mesh.py:113-198) ------------------------------------------------------
    mesh = cantilever(7, 5)
    g["mesh_vertices"] = mesh.vertices
    g["mesh_triangles"] = mesh.triangles
    g["mesh_facets"] = mesh.boundary_facets
    g["mesh_tags"] = mesh.facet_tags
    g["mesh_diameter_7x5"] = np.array([mesh_diameter(mesh)])
    odd = build_rect_mesh((-0.3, 0.1, 1.7, 1.3), 13, 9)
    g["odd_vertices"] = odd.vertices

    # -- operator, material, Dirichlet (fem.py, base.py, compliance.py) ---------------
    mesh = cantilever(32, 16)
    space = FunctionSpace(mesh, 2)
    scalar = FunctionSpace(mesh, 1)
    phi = LevelSetField.from_field(scalar.interpolate(phi_fn))
    g["phi_32x16"] = phi.values
    g["h_32x16"] = np.array([phi.h])
    g["chi_32x16"] = phi.indicator_quad()
    a_q = MaterialIndicator(1.0, ERSATZ).at_quad(phi)
    K = space.assemble_matrix(elasticity_matrix(space, a_q, LAME))
    rng = np.random.default_rng(42)
    u = rng.standard_normal((3, space.dof_count))
    g["apply_u"] = u
    g["apply_Ku"] = np.stack([K @ x for x in u])
    bc = DirichletSet.on_tags(space, 1)
    g["bc_dofs"] = bc.dofs
    elim = apply_dirichlet(SparseSystem(K, np.zeros(space.dof_count)), bc).matrix
    g["apply_Keu"] = np.stack([elim @ x for x in u])
    g["diag_elim"] = elim.diagonal()

    # -- compliance model pieces (compliance.py:37-139) --------------------------------
    bil = BilinearSpec(mass_weight=1.0, stiffness_weight=1e-2)
    model = ComplianceModel(mesh, 1, 2, (0.0, -1.0), 1.0, lame=LAME, bilinear=bil)
    model.material = MaterialIndicator(1.0, ERSATZ)
    problems = model.pde(phi)
    g["load_vector"] = problems[0].rhs
    states = [solve_problem(p) for p in problems]
    g["state_u"] = states[0].values
    J = model.cost(phi, states)
    C = model.constraint(phi, states)
    g["J"] = np.array([J])
    g["C"] = np.asarray(C)
    adjoints = model.adjoint(phi, states)
    cost_pair, cons = model.derivative(phi, states, adjoints)
    g["S1_cost"] = cost_pair.s1(space)
    lam = np.array([0.37])
    pair = combine_derivatives(cost_pair, cons, lam)
    solver = VelocitySolver(bil, space)
    vec = solver._derivative_vector(pair)
    g["velocity_vec"] = vec
    res = solver.solve(pair)
    g["theta"] = res.theta.values
    g["form_value"] = np.array([res.form_value])
    g["derivative"] = np.array([res.derivative])

    # velocity forms with the optional terms (velocity.py:32-127)
    for name, spec in {
        "normal": BilinearSpec(mass_weight=0.1, stiffness_weight=1.0, boundary_normal_penalty=1e4),
        "dirichlet": BilinearSpec(stiffness_weight=1.0, zero_dirichlet=True),
        "frozen": BilinearSpec(mass_weight=1.0, stiffness_weight=0.5,
                               frozen_subdomain=lambda p: p[:, 0] > 1.6, frozen_penalty=1e2),
    }.items():
        s = VelocitySolver(spec, space)
        r = s.solve(pair)
        g[f"theta_{name}"] = r.theta.values
        g[f"form_value_{name}"] = np.array([r.form_value])
        g[f"form_apply_{name}"] = s.form_matrix @ u[0]

    # two identical loads double J (test_models.py:175-187) -- batched path check
    plus = CompliancePlusModel(mesh, 1, [((0.0, -1.0), 2), ((0.0, -2.0), 2)], 1.0, lame=LAME,
                               bilinear=bil)
    plus.material = MaterialIndicator(1.0, ERSATZ)
    pst = [solve_problem(p) for p in plus.pde(phi)]
    g["plus_J"] = np.array([plus.cost(phi, pst)])
    g["plus_states"] = np.stack([s.values for s in pst])

    # body force load (fem.py:419-425)
    f_q = np.broadcast_to(np.array([0.0, -1.0]), (mesh.num_triangles, 3, 2))
    g["body_force_vector"] = space.assemble_vector(vector_load(space, f_q))

    # -- PPL (ppl.py:47-114) -------------------------------------------------------------
    st = ppl_init(1)
    cs = [1.55, 1.3, 1.1, 0.95, 1.02, 0.99, 1.0]
    rows = []
    for c in cs:
        st = ppl_update(st, [c])
        rows.append([st.z[0], st.lam[0], st.mu[0], st.delta, lagrangian_value(2.0, [c], st)])
    g["ppl_table"] = np.array(rows)
    g["ppl_inputs"] = np.array(cs)

    # -- adaptive_time with the host RNG (driver.py:121-143) -----------------------------
    params = ldriver.RunParams()
    r = np.random.default_rng(1)
    at = [ldriver.adaptive_time(b, params, r) for b in (0.2, 0.05, 3.0, 1e-9, 17.0, 0.6)]
    g["adaptive_btt"] = np.array([0.2, 0.05, 3.0, 1e-9, 17.0, 0.6])
    g["adaptive_out"] = np.array(at, dtype=float)

    # -- the reference's own level-set scheme (levelset.py:137-216) ----------------------
    from lsopt.levelset import reinitialize, transport

    sq = build_rect_mesh((0.0, 0.0, 1.0, 1.0), 24, 20)
    s1sp, s2sp = FunctionSpace(sq, 1), FunctionSpace(sq, 2)
    phi_sq = LevelSetField.from_field(
        s1sp.interpolate(lambda p: np.hypot(p[:, 0] - 0.45, p[:, 1] - 0.55) - 0.3 + 0.05 * np.sin(5 * p[:, 0])))
    th_sq = s2sp.interpolate(lambda p: np.stack([np.sin(np.pi * p[:, 0]) * np.cos(2 * p[:, 1]),
                                                 0.3 + p[:, 0] * p[:, 1]], axis=1))
    g["ls_phi"] = phi_sq.values
    g["ls_theta"] = th_sq.values
    g["ls_transport"] = transport(phi_sq, th_sq, 0.03, 8, smooth=False).values
    g["ls_transport_smooth"] = transport(phi_sq, th_sq, 0.03, 8, smooth=True).values
    g["ls_reinit"] = reinitialize(LevelSetField(FemField(s1sp, 3.0 * phi_sq.values), phi_sq.h),
                                  8, 0.1).values

    # -- a full reference run() on the cfg1 geometry at 40x20 (driver.py:211-298) -----
    from lsopt.driver import RunParams, run

    rules = [(1, lambda p: p[:, 0] < 1e-12),
             (2, lambda p: (p[:, 0] > 2.0 - 1e-12) & (p[:, 1] >= 0.45) & (p[:, 1] <= 0.55))]
    m40 = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 40, 20, rules)
    model40 = ComplianceModel(m40, 1, 2, (0.0, -1.0), 1.0, lame=LAME, bilinear=bil)
    model40.material = MaterialIndicator(1.0, ERSATZ)
    phi40 = LevelSetField.from_field(FunctionSpace(m40, 1).interpolate(phi_fn))
    params = RunParams(niter=12, start_to_check=12, reinit_step=5, reinit_pars=(8, 0.1))
    _, hist = run(model40, phi40, params, timing=False)
    g["run_cost"] = np.array([r.cost for r in hist])
    g["run_constraint"] = np.array([float(r.constraint[0]) for r in hist])
    g["run_lagrangian"] = np.array([r.lagrangian for r in hist])
    g["run_t_end"] = np.array([r.t_end for r in hist])
    g["run_steps"] = np.array([r.steps for r in hist])
    g["run_form_value"] = np.array([r.form_value for r in hist])

    # -- output formats (output.py:23-124): bytes of the reference writers ---------------
    import tempfile

    from lsopt.output import write_history_csv, write_vtk

    with tempfile.TemporaryDirectory() as tmp:
        write_history_csv(os.path.join(tmp, "h.csv"), hist)
        g["run_history_csv"] = np.array(open(os.path.join(tmp, "h.csv")).read())
        m32 = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 3, 2)
        f1 = FunctionSpace(m32, 1).interpolate(lambda p: np.sin(p[:, 0]) - p[:, 1] / 3.0)
        f2 = FunctionSpace(m32, 2).interpolate(lambda p: np.stack([p[:, 0] / 7.0, -p[:, 1]], 1))
        write_vtk(m32, {"phi": f1, "theta": f2}, os.path.join(tmp, "m.vtk"))
        g["vtk_text"] = np.array(open(os.path.join(tmp, "m.vtk")).read())

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, sum(v.nbytes for v in g.values()) / 1e6, "MB raw")


if __name__ == "__main__":
    main()
