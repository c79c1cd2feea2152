"""Outer optimisation loop (oracle; test infrastructure only).

Restates reference ``driver.py:121-298`` -- ``adaptive_time`` (``:121-143``),
``stopping_check`` (``:146-166``) and ``run`` (``:211-298``) with the same
loop order: states (warm-started, ``:238-249``) -> adjoints (-2u, closed
form) -> J, C -> PPL update -> record -> stop? -> S1 -> velocity -> descent
guards (``:273-285``) -> adaptive horizon (host RNG ``default_rng(seed)``,
uniform then normal, ``:137-141``) -> transport -> reinit on
``(it+1) % reinit_step == 0`` (``:288``) -- except that transport and
reinitialisation are the explicit schemes of ``oracle.levelset``.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from . import fem, levelset, model as mdl

BTT_FLOOR = 1e-12


@dataclass(frozen=True)
class Params:
    niter: int = 100
    dfactor: float = 1e-2
    lv_time: tuple = (1e-3, 1e-1)
    lv_iter: tuple = (8, 16)
    smooth: bool = False
    reinit_step: object = None
    reinit_pars: tuple = (8, 1e-1)
    start_to_check: int = 30
    ctrn_tol: float = 1e-2
    lgrn_tol: float = 1e-2
    cost_tol: float = 1e-2
    prev: int = 10
    random_pars: tuple = (1, 0.05)
    scheme: str = "explicit"  # level-set update: "explicit" (north star) or "pg" (reference)


def adaptive_time(btt, params, rng):
    t_min, t_max = params.lv_time
    s_min, s_max = params.lv_iter
    spread = float(params.random_pars[1])
    t_end = params.dfactor / max(btt, BTT_FLOOR)
    if spread > 0.0:
        t_end *= rng.uniform(1.0 - spread, 1.0 + spread)
    t_end = min(max(t_end, t_min), t_max)
    s_hat = (s_max - s_min) * ((t_end - t_min) / (t_max - t_min)) ** (1.0 / 6.0) + s_min
    if spread > 0.0:
        s_hat = rng.normal(s_hat, spread * s_hat)
    return t_end, int(round(min(max(s_hat, s_min), s_max)))


def stopping_check(history, params, has_constraints):
    if not history:
        return False
    cur = history[-1]
    if cur["iteration"] <= params.start_to_check:
        return False
    window = history[max(len(history) - 1 - params.prev, 0): len(history) - 1]
    if not window:
        return False
    if has_constraints:
        if not cur["ctrn_err"] < params.ctrn_tol:
            return False
        swing = max(abs(cur["lagrangian"] - r["lagrangian"]) for r in window)
        return swing < params.lgrn_tol * abs(cur["lagrangian"])
    swing = max(abs(cur["cost"] - r["cost"]) for r in window)
    return swing < params.cost_tol * abs(cur["cost"])


def run(model, velocity, phi0, params, h, rtol=fem.CG_RTOL, on_record=None):
    """Returns (phi, history); history rows are dicts with the reference's
    IterationRecord fields plus the discrete counters (CG iterations, substeps)."""
    grid = model.grid
    history = []
    if params.niter == 0:
        return phi0, history
    rng = np.random.default_rng(int(params.random_pars[0]))
    ppl = mdl.ppl_init(1)
    phi = np.asarray(phi0, dtype=float).copy()
    warm = None
    for it in range(params.niter):
        states, iters = model.solve_states(phi, warm, rtol=rtol)
        warm = [u.copy() for u in states]
        cost = model.cost(phi, states)
        cvals = np.array([model.constraint(phi)])
        ppl = mdl.ppl_update(ppl, cvals)
        rec = dict(iteration=it, cost=cost, constraint=cvals.copy(),
                   lagrangian=mdl.lagrangian(cost, cvals, ppl),
                   ctrn_err=float(np.max(np.abs(cvals - 1.0))), multipliers=ppl.lam.copy(),
                   t_end=0.0, steps=0, form_value=0.0, cg_iters=iters,
                   nsub_transport=0, nsub_reinit=0)
        history.append(rec)
        if stopping_check(history, params, True):
            if on_record:
                on_record(rec, phi)
            return phi, history
        s1 = model.s1_combined(phi, states, float(ppl.lam[0]))
        vec = mdl.derivative_vector(model.space, s1=s1)
        theta, btt, dj = velocity.solve(vec)
        slack = 1e-12 * (1.0 + abs(btt))
        if btt < -slack or dj > slack:
            raise fem.SolverError(f"velocity solve lost descent: dJ={dj:.3e}, B={btt:.3e}", dj)
        if abs(dj + btt) > 1e-8 * (1.0 + abs(btt)):
            raise fem.SolverError("velocity derivative identity broke", dj + btt)
        t_end, steps = adaptive_time(btt, params, rng)
        if params.scheme == "pg":
            phi, nt = levelset.transport_pg(grid, phi, theta, t_end, steps, params.smooth, h), steps
        else:
            phi, nt = levelset.transport(grid, phi, theta, t_end, steps, params.smooth, h)
        rec["nsub_transport"] = nt
        if params.reinit_step is not None and (it + 1) % params.reinit_step == 0:
            iters_r, t_final = params.reinit_pars
            if params.scheme == "pg":
                phi, nr = levelset.reinitialize_pg(grid, phi, int(iters_r), float(t_final), h), int(iters_r)
            else:
                phi, nr = levelset.reinitialize(grid, phi, int(iters_r), float(t_final), h)
            rec["nsub_reinit"] = nr
        rec["t_end"], rec["steps"], rec["form_value"] = t_end, steps, btt
        if on_record:
            on_record(rec, phi)
    return phi, history
