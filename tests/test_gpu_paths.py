"""The ways a 2D PCG chunk can run give the same solutions: the 16-CTA cluster
kernel and the cooperative persistent kernel (small systems), CUDA-graph
replays and direct launches of the per-launch single pass, and its stored-q
variant (LSG_PCG2D_RQ=0) beside the default recompute-q pass -- including
right-hand sides that converge in the middle of a chunk and a zero right-hand
side.  Each path runs in its own process because the switches are read once
per process.  Needs a B200."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
from paper_2601_05709_b200 import DirichletSet, ElasticityOperator, FunctionSpace, build_rect_mesh
from paper_2601_05709_b200.fem import solve_batched
mesh = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 48, 24, [(1, lambda p: p[:, 0] < 1e-12)])
space = FunctionSpace(mesh, 2)
rng = np.random.default_rng(3)
phi = torch.as_tensor(rng.standard_normal(mesh.num_vertices), device="cuda")
op = ElasticityOperator(space, phi, (0.33, 0.38), 1e-3, DirichletSet.on_tags(space, 1))
b = rng.standard_normal((3, space.dof_count))
b[1] *= 1e-3          # converges at a different iteration
b[2] = 0.0            # zero right-hand side: x = 0, no iterations
bc = DirichletSet.on_tags(space, 1).dofs
b[:, bc] = 0.0
x, it = solve_batched(op, torch.as_tensor(b, device="cuda"), rtol=1e-10)
np.save(sys.argv[1], x.cpu().numpy())
# a 2x1-cell system: CG ends in ~n steps and its last x += alpha p is O(|x|), so a
# pending update applied with the wrong direction buffer shows at once
tiny = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 2, 1, [(1, lambda p: p[:, 0] < 1e-12)])
ts = FunctionSpace(tiny, 2)
top = ElasticityOperator(ts, torch.as_tensor(rng.standard_normal(tiny.num_vertices) - 0.2, device="cuda"),
                         (0.33, 0.38), 1e-3, DirichletSet.on_tags(ts, 1))
tb = rng.standard_normal((3, ts.dof_count)) * np.array([[1.0], [1e-2], [1e3]])
tb[:, DirichletSet.on_tags(ts, 1).dofs] = 0.0
tx, tit = solve_batched(top, torch.as_tensor(tb, device="cuda"), rtol=1e-12)
np.save(sys.argv[1] + ".tiny.npy", tx.cpu().numpy())
np.save(sys.argv[1] + ".tinyres.npy", (torch.as_tensor(tb, device="cuda") - top.apply(tx)).norm(dim=1).cpu().numpy()
        / np.linalg.norm(tb, axis=1))
print(json.dumps([int(v) for v in it.cpu()]))
"""


def run_path(tmp_path, name, env):
    out = tmp_path / f"{name}.npy"
    script = tmp_path / "solve.py"
    script.write_text(SCRIPT % {"root": ROOT})
    full = dict(os.environ, **env)
    res = subprocess.run([sys.executable, str(script), str(out)], env=full, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    tiny = (np.load(str(out) + ".tiny.npy"), np.load(str(out) + ".tinyres.npy"))
    return np.load(out), json.loads(res.stdout.strip().splitlines()[-1]), tiny


def test_pcg_paths_agree(tmp_path):
    xp, itp, tp = run_path(tmp_path, "persistent", {})
    xg, itg, tg = run_path(tmp_path, "graph", {"LSG_PCG2D_PERSISTENT": "0"})
    xd, itd, td = run_path(tmp_path, "direct", {"LSG_PCG2D_PERSISTENT": "0", "LSG_NO_GRAPHS": "1"})
    xq, itq, tq = run_path(tmp_path, "storedq", {"LSG_PCG2D_PERSISTENT": "0", "LSG_PCG2D_RQ": "0"})
    # small systems default to the 16-CTA cluster kernel; this is the cooperative one
    xc, itc, tc = run_path(tmp_path, "coop", {"LSG_PCG2D_CLUSTER": "0"})
    for x, res in (tp, tg, td, tq, tc):  # every path meets the stopping rule in the true residual
        assert (res <= 1e-10).all(), res
    assert np.linalg.norm(tp[0] - tg[0]) <= 1e-10 * np.linalg.norm(tg[0])
    assert itp[2] == itg[2] == itd[2] == 0 and not xp[2].any() and not xg[2].any()
    assert itg == itd and np.array_equal(xg, xd)  # same kernels, same order: bitwise
    # recomputed q_{i-1} is bit-identical to the stored one; only the grouping of
    # the per-thread partial sums differs (28- vs 30-column strips)
    assert itq[2] == 0 and not xq[2].any()
    for r in range(2):
        assert abs(itq[r] - itg[r]) <= max(2, itg[r] // 50)
        assert np.linalg.norm(xq[r] - xg[r]) <= 1e-8 * np.linalg.norm(xg[r])
    assert itc[2] == 0 and not xc[2].any()
    for r in range(2):  # cluster vs cooperative: same pass, other reduction grouping
        assert abs(itc[r] - itp[r]) <= max(2, itp[r] // 50)
        assert np.linalg.norm(xc[r] - xp[r]) <= 1e-8 * np.linalg.norm(xp[r])
    for r in range(2):
        assert itp[r] > 10 and abs(itp[r] - itg[r]) <= max(2, itp[r] // 20)
        assert np.linalg.norm(xp[r] - xg[r]) <= 1e-8 * np.linalg.norm(xg[r])


SWEEP = r"""
import sys
sys.path.insert(0, %(root)r)
sys.path.insert(0, %(tests)r)
import test_gpu_shapes as t
for n in t.SHAPES_2D + [(7, 40), (33, 61)]:
    t.test_shapes_2d(n)
print("ok")
"""


def test_shape_sweep_graph_paths(tmp_path):
    """The 2D grid-shape sweep (state PCG, velocity CG) with the persistent
    kernel off, so every solve runs the per-launch single pass: the default
    recompute-q pass (28-column strips, two halo rows per segment) at both
    prefetch depths and the stored-q pass, on grids around every tile edge and with many row segments."""
    script = tmp_path / "sweep.py"
    script.write_text(SWEEP % {"root": ROOT, "tests": os.path.join(ROOT, "tests")})
    for env in ({"LSG_PCG2D_PERSISTENT": "0"}, {"LSG_PCG2D_PERSISTENT": "0", "LSG_RQ_AHEAD": "2"},
                {"LSG_PCG2D_PERSISTENT": "0", "LSG_RQ_AHEAD": "3"},
                {"LSG_PCG2D_PERSISTENT": "0", "LSG_PCG2D_RQ": "0"}):
        res = subprocess.run([sys.executable, str(script)], env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=900)
        assert res.returncode == 0 and res.stdout.strip().endswith("ok"), (env, res.stderr[-3000:])


SCRIPT3D = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
from paper_2601_05709_b200 import DirichletSet, ElasticityOperator, FunctionSpace, build_box_mesh
from paper_2601_05709_b200.fem import solve_batched
mesh = build_box_mesh((0.0, 0.0, 0.0, 2.0, 1.0, 1.0), (12, 6, 6), [(1, lambda p: p[:, 0] < 1e-12)])
space = FunctionSpace(mesh, 3)
rng = np.random.default_rng(5)
phi = torch.as_tensor(rng.standard_normal(mesh.num_vertices) - 0.2, device="cuda")
bc = DirichletSet.on_tags(space, 1)
op = ElasticityOperator(space, phi, (0.576923, 0.384615), 1e-3, bc)
b = rng.standard_normal((5, space.dof_count)) * np.array([[1.0], [1e-2], [1e3], [0.0], [1.0]])
b[:, bc.dofs] = 0.0
x, it = solve_batched(op, torch.as_tensor(b, device="cuda"), rtol=1e-10)
np.save(sys.argv[1], x.cpu().numpy())
print(json.dumps([int(v) for v in it.cpu()]))
"""


def test_pcg3d_two_streams_agree(tmp_path):
    """3D batched PCG split over two streams (default) vs one stream: an odd
    batch with a zero right-hand side and right-hand sides that converge at
    different iterations gives the same solutions."""
    script = tmp_path / "solve3d.py"
    script.write_text(SCRIPT3D % {"root": ROOT})
    out = {}
    for name, env in (("two", {}), ("one", {"LSG_PCG3D_STREAMS": "1"})):
        res = subprocess.run([sys.executable, str(script), str(tmp_path / f"{name}.npy")],
                             env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        out[name] = (np.load(tmp_path / f"{name}.npy"), json.loads(res.stdout.strip().splitlines()[-1]))
    (x2, it2), (x1, it1) = out["two"], out["one"]
    assert it2[3] == it1[3] == 0 and not x2[3].any()
    for r in (0, 1, 2, 4):
        assert it1[r] > 10 and abs(it1[r] - it2[r]) <= max(2, it1[r] // 50)
        assert np.linalg.norm(x2[r] - x1[r]) <= 1e-8 * np.linalg.norm(x1[r])
