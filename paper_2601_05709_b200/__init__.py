"""B200-native (sm_100a) core of FormOpt's level-set shape-optimisation loop.

Drop-in for the hot path of the reference package ``lsopt`` 0.1.0
(``/root/reference/pkg/src/lsopt``): the same public entry points
(``run``, ``RunParams``, ``solve_concurrent``, ``transport``,
``reinitialize``, ``VelocitySolver``, the compliance models ...), with the
arithmetic in hand-written fp64 CUDA kernels (``liblsgpu.so``, C ABI in
``include/lsgpu.h``) and PyTorch used only to hold device memory and streams.
There is no CPU fallback: without the library or a CUDA device every
operation raises.
"""

from .driver import (IterationRecord, RunParams, adaptive_time, run, solve_concurrent,
                     stopping_check)
from .errors import ConfigError, NewtonError, SolverError
from .fem import (DirichletSet, ElasticityOperator, FemField, FunctionSpace, H1Operator, LaplaceOperator,
                  LinearProblem, solve_batched, solve_linear)
from .levelset import InitialLevelSpec, LevelSetField, initial_level, reinitialize, transport
from .mesh import (BoxMesh, RectMesh, build_box_mesh, build_rect_mesh, mesh_diameter,
                   tag_boundary)
from .models import (ComplianceModel, CompliancePlusModel, HeatModel, HeatPlusModel, HeatTerm,
                     InverseElasticityModel, MeasurementPair, dirichlet_extension,
                     generate_measurements)
from .ppl import combine_derivatives, lagrangian_value, ppl_init, ppl_update
from .velocity import BilinearSpec, DerivativePair, VelocityResult, VelocitySolver

__all__ = [
    "ConfigError", "NewtonError", "SolverError", "RunParams", "IterationRecord", "adaptive_time",
    "stopping_check", "solve_concurrent", "run", "RectMesh", "BoxMesh", "build_rect_mesh",
    "build_box_mesh", "mesh_diameter", "tag_boundary", "InitialLevelSpec", "LevelSetField",
    "initial_level", "reinitialize", "transport", "FunctionSpace", "FemField", "DirichletSet",
    "ElasticityOperator", "H1Operator", "LaplaceOperator", "LinearProblem", "solve_linear", "solve_batched",
    "ComplianceModel", "CompliancePlusModel", "HeatModel", "HeatPlusModel", "HeatTerm", "InverseElasticityModel",
    "MeasurementPair", "dirichlet_extension", "generate_measurements", "BilinearSpec", "DerivativePair", "VelocityResult",
    "VelocitySolver", "combine_derivatives", "lagrangian_value", "ppl_init", "ppl_update",
]

__version__ = "0.1.0"
