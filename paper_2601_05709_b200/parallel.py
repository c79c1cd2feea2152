"""Load-case sharding across GPUs.

The batched state solve is embarrassingly parallel over load cases; the one
real exchange of the loop is the sum over load cases of the compliance J and
of the contracted cost-derivative vector (``compliance.py:111-139``).  With
``ShardedCompliance`` each rank (one process per GPU, ``torch.distributed``
over NCCL / NVLink) keeps the full grid and phi, solves only its share of
the load cases as one batched PCG, and all-reduces

* J (one double; the volume is identical on every rank and is not reduced),
* vec_cost (d N doubles, 4.2 MB at cfg2 -- a few microseconds over NVLink 5),

once per optimisation iteration.  The velocity solve, transport and
reinitialisation then run redundantly on every rank from identical inputs
with deterministic kernels, so phi stays bitwise identical across ranks and
no further collective is needed.

The split and the reduction bookkeeping are plain host logic
(``shard_loads``, ``reduce_partials``) so they are tested with the gloo
backend on CPU (tests/test_parallel.py).
"""

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigError
from .models.compliance import CompliancePlusModel, ComplianceModel

__all__ = ["shard_loads", "reduce_partials", "ShardedCompliance"]


def shard_loads(k, rank, world):
    """Contiguous block of load-case indices owned by ``rank`` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of {world}")
    base, extra = divmod(k, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def reduce_partials(J_local, vec_local, group=None):
    """Sum the per-rank compliance and cost-derivative vector (in place on vec_local)."""
    t = torch.tensor([float(J_local)], dtype=torch.float64, device=vec_local.device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(vec_local, op=dist.ReduceOp.SUM, group=group)
    return float(t.item()), vec_local


class ShardedCompliance(CompliancePlusModel):
    """A compliance model whose load cases are split across the ranks of ``group``.

    Same contract as ``CompliancePlusModel``; ``pde`` returns this rank's
    problems only, ``cost`` / ``derivative`` return the global (all-rank)
    quantities.  A rank may own zero load cases (k < world).
    """

    def __init__(self, model: ComplianceModel, group=None):
        self.__dict__.update(model.__dict__)
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.owned = shard_loads(int(model.load_vectors.shape[0]), rank, world)
        self._all_loads = model.load_vectors
        self._loads = model.load_vectors[self.owned] if self.owned else model.load_vectors[:0]
        self._cache_key = None

    def pde(self, phi):
        return super().pde(phi)

    def _evaluate(self, phi, states):
        key = (id(phi), tuple(id(u) for u in states))
        if self._cache_key == key:
            return self._cache
        if states:
            J, vol, vc, vv, u = super()._evaluate(phi, states)
        else:  # no local load case: contribute zeros, still compute the volume terms
            from .fem import FemField
            zero = FemField(self.space, torch.zeros(self.space.dof_count, dtype=torch.float64, device="cuda"))
            J, vol, vc, vv, u = super()._evaluate(phi, [zero])
            J = 0.0
            vc = torch.zeros_like(vc)
        J, vc = reduce_partials(J, vc, self.group)
        self._cache_key = key
        self._cache = (J, vol, vc, vv, u)
        return self._cache
