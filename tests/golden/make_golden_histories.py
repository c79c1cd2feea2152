"""Oracle histories of the BASELINE configs at (or near) their own size -- the parity
fixtures for the north star's "J/C history within 1e-4 over the config's iteration
count" (VERDICT round 1 "pin parity at config size").

    python tests/golden/make_golden_histories.py cfg3            # full 96x48x48, 30 it
    python tests/golden/make_golden_histories.py cfg2_half       # 512x128, all 40 it
    python tests/golden/make_golden_histories.py cfg2_full3      # 1024x256, first 3 it
    python tests/golden/make_golden_histories.py cfg5_half       # 96x48x48, 4 loads, 20 it
    python tests/golden/make_golden_histories.py cfg5_full1      # 192x96x96, 4 loads, first iteration
    python tests/golden/make_golden_histories.py cfg5_full3      # 192x96x96, 4 loads, first 3 iterations

Each writes tests/golden/oracle_<name>.npz.  CPU only (tens of minutes to hours:
the oracle is scipy CSR + scipy ``cg``, single-threaded per solve).  The k load
cases of one iteration are solved in k forked processes (the solves are
independent, exactly as the reference's ``task_parallel`` mode, driver.py:185-194);
the results are identical to the serial oracle.  The 3D velocity form is solved
by Jacobi-CG to 1e-14 instead of SuperLU (``oracle.model.Velocity(direct=False)``:
the 3D LU fill is out of reach at these sizes).  The oracle itself is pinned to
the reference's own run() history in 2D (tests/test_oracle.py); the 3D pieces
are restatements (property-pinned).
"""

import os

# one BLAS thread per process: the oracle's scipy cg is a chain of small BLAS
# calls, and threaded OpenBLAS on a shared host makes each ~50x slower
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import multiprocessing as mp  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import cases as ocases, driver as odriver, fem as ofem  # noqa: E402
from paper_2601_05709_b200 import configs  # noqa: E402

# name -> (config, scale, niter, direct velocity LU)
JOBS = {
    "cfg3": ("cfg3", 1, 30, False),
    "cfg2_half": ("cfg2", 2, 40, True),
    "cfg2_full3": ("cfg2", 1, 3, True),
    "cfg5_half": ("cfg5", 2, 20, False),
    # full size: the oracle assembles its matrices 400k tets at a time
    # (Space.assemble_matrix_by_parts); ~20 GB resident, ~2 h for one iteration
    "cfg5_full1": ("cfg5", 1, 1, False),
    "cfg5_full3": ("cfg5", 1, 3, False),  # warm-started solves on a transported level set (~2 h)
    "cfg5_full5": ("cfg5", 1, 5, False),  # ... through the first reinitialisation (~3 h)
}

_SYSTEMS = None


def _solve_one(args):
    k, x0, rtol = args
    A, b = _SYSTEMS[k]
    return ofem.jacobi_pcg(A, b, x0=x0, rtol=rtol)


def parallel_states(model):
    """model.solve_states with the k independent solves in forked processes."""
    def solve_states(phi, warm=None, rtol=ofem.CG_RTOL):
        global _SYSTEMS
        _SYSTEMS = model.eliminated(phi)
        k = len(_SYSTEMS)
        jobs = [(i, None if warm is None else warm[i], rtol) for i in range(k)]
        if k == 1:
            out = [_solve_one(jobs[0])]
        else:
            with mp.get_context("fork").Pool(k) as pool:
                out = pool.map(_solve_one, jobs)
        _SYSTEMS = None
        return [x for x, _ in out], [it for _, it in out]
    return solve_states


def main(name):
    cfg, scale, niter, direct = JOBS[name]
    c = configs.case(cfg, scale=scale)
    c = type(c)(**{**c.__dict__, "niter": niter})
    grid, om, ovel, ophi, oparams, h = ocases.build(c, direct=direct)
    om.solve_states = parallel_states(om)
    t0 = time.time()

    keys = ("cost", "lagrangian", "form_value", "t_end", "steps", "nsub_transport", "nsub_reinit")
    done = []

    def save(rows):
        out = {k: np.array([r[k] for r in rows]) for k in keys}
        out["constraint"] = np.array([r["constraint"][0] for r in rows])
        out["cg_iters"] = np.array([r["cg_iters"] for r in rows])
        out["grid"] = np.array(c.n)
        np.savez_compressed(os.path.join(HERE, f"oracle_{name}.npz"), **out)
        return out

    def on_record(rec, phi):
        print(f"[{name}] it {rec['iteration']:3d}  J={rec['cost']:.10e}  C={rec['constraint'][0]:.10e}  "
              f"cg={sum(rec['cg_iters'])}  steps={rec['steps']}  nsub={rec['nsub_transport']}/"
              f"{rec['nsub_reinit']}  {time.time() - t0:.0f}s", flush=True)
        # every completed iteration is a valid fixture (a run of n iterations is the
        # prefix of a longer one): keep the file current, a long job can be cut short
        done.append(dict(rec))
        save(done)

    _, hist = odriver.run(om, ovel, ophi, oparams, h, on_record=on_record)
    out = save(hist)
    print(name, len(hist), out["cost"][[0, -1]], f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        main(arg)
