"""Multi-process host logic of load-case sharding (gloo, world_size 2, CPU).

Each rank evaluates its share of the load cases of a cfg2-geometry problem
with the CPU oracle and the partial compliance / cost-derivative vectors are
combined with ``paper_2601_05709_b200.parallel.reduce_partials`` over gloo; the
result must equal the unsharded evaluation.  (The GPU kernels are exercised
by the -m gpu suites; this checks the split and the collective bookkeeping.)
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_05709_b200.parallel import reduce_partials, shard_loads


def test_shard_loads_partition():
    for k in range(0, 11):
        for world in range(1, 6):
            parts = [shard_loads(k, r, world) for r in range(world)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(k))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    from oracle import cases as ocases
    from paper_2601_05709_b200 import configs
    c = configs.case("cfg2", scale=16)
    grid, om, _, phi, _, _ = ocases.build(c, velocity=False)
    states, _ = om.solve_states(phi, rtol=1e-10)
    return om, phi, states


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import model as omodel
        om, phi, states = _problem()
        mine = shard_loads(len(states), rank, world)
        sub = [states[i] for i in mine]
        J_local = om.cost(phi, sub) if sub else 0.0
        vec_local = omodel.derivative_vector(om.space, s1=om.s1_cost(phi, sub)) if sub else \
            np.zeros(om.space.dof_count)
        J, vec = reduce_partials(J_local, torch.from_numpy(vec_local.copy()))
        out[rank] = (J, vec.numpy().copy(), mine)
    finally:
        dist.destroy_process_group()


def test_sharded_reduction_matches_unsharded():
    from oracle import model as omodel
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    om, phi, states = _problem()
    J_ref = om.cost(phi, states)
    vec_ref = omodel.derivative_vector(om.space, s1=om.s1_cost(phi, states))
    assert sorted(out[0][2] + out[1][2]) == list(range(len(states)))
    for r in range(world):
        J, vec, _ = out[r]
        assert J == pytest.approx(J_ref, rel=1e-13)
        assert np.linalg.norm(vec - vec_ref) <= 1e-13 * np.linalg.norm(vec_ref)
    # both ranks hold bitwise-identical reduced results (redundant velocity solve input)
    np.testing.assert_array_equal(out[0][1], out[1][1])
