"""Build the oracle's model for a configuration record (oracle; test infrastructure only).

Takes the same plain ``Case`` data the product harness uses
(``paper_2601_05709_b200/configs.py``; duck-typed, not imported here) and
assembles the CPU restatement: Grid + Compliance + Velocity + Params.
"""

import numpy as np

from . import fem
from .driver import Params
from .grid import Grid, level_set_h
from .model import Compliance, Velocity


def build(c, velocity=True, direct=True):
    # tag 1 = clamp; one tag per distinct load patch (first-match tagging)
    rules, tags, seen = [(1, c.fixed)], [], {}
    for _, pred in c.loads:
        if id(pred) not in seen:
            seen[id(pred)] = 2 + len(seen)
            rules.append((seen[id(pred)], pred))
        tags.append(seen[id(pred)])
    grid = Grid(c.lo, c.hi, c.n, rules)
    space = fem.Space(grid, grid.dim)
    clamp = fem.clamp_dofs(space, grid.facets_with_tag(1))
    loads = [fem.boundary_traction_vector(space, grid.facets_with_tag(t), g)
             for (g, _), t in zip(c.loads, tags)]
    if c.body_force is not None:
        bf = fem.body_force_vector(space, c.body_force)
        loads = [v + bf for v in loads] if loads else [bf]
    model = Compliance(grid, c.lame, c.ersatz, clamp, loads, c.volume)
    velocity = (Velocity(grid, mass_weight=c.h1[0], stiffness_weight=c.h1[1], direct=direct)
                if velocity else None)
    phi0 = np.asarray(c.phi0(grid.vertices), dtype=float)
    params = Params(niter=c.niter, start_to_check=c.niter, reinit_step=c.reinit_step,
                    reinit_pars=c.reinit_pars)
    return grid, model, velocity, phi0, params, level_set_h(grid)
