"""CPU oracle for the level-set compliance loop -- TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference algorithm
(``/root/reference/pkg/src/lsopt``, ``lsopt`` 0.1.0) for the north-star hot
path.  Most of it is written from the reference's formulas; the one exception
is the reference's own Crank-Nicolson Petrov-Galerkin transport / PG-AB2
reinitialisation (``levelset.transport_pg`` / ``reinitialize_pg`` and their
helpers, ``levelset.py:177-287`` here), which follows the reference's code
(``levelset.py:109-278``) closely on purpose: it has to reproduce that
scheme's floating-point behaviour to pin the device PG scheme.  It exists to
check the CUDA path, never to stand in for it: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product package
``paper_2601_05709_b200`` never imports it and fails loudly when its CUDA
library is missing.

Pinning
-------
* 2D mesh / FEM / compliance / velocity / PPL / driver pieces are pinned
  against the reference itself: ``tests/golden/make_golden.py`` imports the
  reference (from ``/root/reference/pkg/src``, available only in the build
  container) and commits small golden vectors that ``tests/test_oracle.py``
  checks the restatement against.
* The explicit upwind transport / Godunov reinitialisation (north star (4))
  and all 3D pieces have no reference implementation (the reference is 2D
  only, ``fem.py:63-64``; its level-set update is Crank-Nicolson
  Petrov-Galerkin, ``levelset.py:137-216``).  Those restatements are pinned
  by the reference's scheme-agnostic property tests
  (``tests/test_levelset.py:155-286`` of the reference) re-run on the oracle,
  and, for 3D, by dimension-generic identities (rigid-motion kernel, patch
  tests, symmetry).  Their parity status is "restated, property-pinned".

Modules
-------
grid       structured rectangle / box meshes (mesh.py:113-198 restated, + Kuhn tets)
fem        P1 spaces, element kernels, CSR assembly, Dirichlet elimination,
           Jacobi-PCG via scipy ``cg`` (fem.py:56-466 restated, d = 2, 3)
levelset   explicit upwind transport + Godunov reinitialisation (restated spec),
           and the reference's CN/PG scheme (levelset.py:109-278)
model      compliance / heat / inverse models (models/*.py restated), the H1
           velocity form and solve (velocity.py:32-159; SuperLU, or Jacobi-CG to
           1e-14 for large 3D fixtures), PPL recursion (ppl.py:47-114)
driver     outer loop (driver.py:121-298 restated)
cases      the BASELINE configurations assembled for the oracle
"""
