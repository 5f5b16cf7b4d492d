"""One instance split over ranks (config C4's multi-GPU split; partition.py).

A k-part deferred-schedule averaging solve must be BIT-IDENTICAL to the
one-GPU/one-process solve of the whole instance: every per-diagram operation
is local, and boundary variables are averaged from an exact exchange buffer
in global copy order.  Checked:

* CPU, world size 2 over gloo: two processes, each owning half the diagrams
  (oracle-backed engine, tests/partition_engines.py) == the oracle's own
  deferred mma-only solve of the whole instance;
* CPU, k = 2, 3, 4 logical parts in one process (LoopbackComm): same;
* GPU, k = 2 and 4 logical parts on one B200 (DeviceEngine, the product
  kernels incl. dm_dfr_boundary_*) == qn.solve(mode="mma-only",
  mma_schedule="deferred") of the whole instance, bounds and duals.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_08230_b200.config import SolveConfig
from paper_2310_08230_b200.partition import DistComm, LoopbackComm, PartitionedSolver, plan_partition, scatter_duals

CFG = SolveConfig(mode="mma-only", mma_schedule="deferred", max_iterations=25)


def _instance(name):
    from bench import build_instance

    if name in ("tetra", "icosa"):
        from paper_2310_08230_b200 import product_space as ps
        from paper_2310_08230_b200.ilp import IlpInstance

        M, N, fm, fn = ps.synthetic_pair(name, 0)
        p = ps.build_product_space(M, N, fm, fn)
        return IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, 128)
    return build_instance(name, 0)


def _oracle_reference(inst):
    from oracle import model, solver

    f = inst.flat
    oi, of = model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts,
                                   {k: getattr(f, k) for k in ("bdd_layer_lo", "layer_node_lo", "layer_var",
                                                               "layer_bdd", "zero_t", "one_t", "proc_ptr",
                                                               "proc_layers")})
    st, rec, stop = solver.solve(oi, mode="mma-only", max_iterations=CFG.max_iterations, dot="chunked", flat=of,
                                 schedule="deferred", damping=CFG.mma_damping)
    return [r[2] for r in rec], st.lam, stop


@pytest.mark.parametrize("name", ["icosa", "c1"])
def test_plan_covers_every_copy_once(name):
    inst = _instance(name)
    f = inst.flat
    for k in (1, 2, 4, 8):
        plan = plan_partition(inst, k)
        assert np.array_equal(np.sort(plan.bdd_order), np.arange(f.num_bdds))
        assert sum(len(p.layers) for p in plan.parts) == f.num_layers
        seen = np.zeros(f.num_layers, int)
        slots = np.zeros(plan.slots, int)
        for p in plan.parts:
            np.add.at(seen, p.layers[p.local_layers], 1)
            np.add.at(seen, p.layers[p.b_layer], 1)
            np.add.at(slots, p.b_slot, 1)
            assert np.all(p.b_lo <= p.b_slot) and np.all(p.b_slot < p.b_hi)
            assert np.array_equal(p.lam0, inst.costs[f.layer_var[p.layers]] / f.constraint_counts[f.layer_var[p.layers]])
        assert np.all(seen == 1)  # every copy averaged exactly once, locally or through the buffer
        assert np.all(slots == 1)  # every boundary slot has exactly one writer
        if k == 1:
            assert plan.slots == 0


@pytest.mark.parametrize("k", [2, 3, 4])
def test_loopback_partitioned_solve_matches_whole_oracle(k):
    from tests.partition_engines import OracleEngine

    inst = _instance("icosa")
    plan = plan_partition(inst, k)
    assert plan.slots > 0
    res = PartitionedSolver(plan, [OracleEngine(p) for p in plan.parts], LoopbackComm(), CFG).solve()
    bounds, lam, stop = _oracle_reference(inst)
    assert res.bounds == bounds and res.stop_reason == stop
    assert scatter_duals(plan, res.lam_parts, inst.flat.num_layers).tobytes() == lam.tobytes()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.partition_engines import OracleEngine

        inst = _instance("icosa")
        plan = plan_partition(inst, world)
        comm = DistComm([p.table.num_bdds for p in plan.parts])
        res = PartitionedSolver(plan, [OracleEngine(plan.parts[rank])], comm, CFG).solve()
        lams = DistComm([p.table.num_layers for p in plan.parts]).allgather_cat([res.lam_parts[0]])[0]
        pieces = torch.split(lams, [p.table.num_layers for p in plan.parts])
        lam = scatter_duals(plan, list(pieces), inst.flat.num_layers)
        out[rank] = (res.bounds, res.stop_reason, lam.tobytes(), plan.slots)
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo_partitioned_solve_matches_whole_oracle():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    bounds, lam, stop = _oracle_reference(_instance("icosa"))
    for r in range(world):
        assert out[r][0] == bounds and out[r][1] == stop
        assert out[r][2] == lam.tobytes()
        assert out[r][3] > 0  # the split really has boundary variables


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c3", "c4"])
@pytest.mark.parametrize("k", [2, 4])
def test_gpu_logical_partitions_match_one_gpu_solve(name, k):
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.partition import DeviceEngine

    inst = _instance(name)
    whole = qn.solve(inst, CFG, device="cuda:0")
    plan = plan_partition(inst, k)
    res = PartitionedSolver(plan, [DeviceEngine(p, "cuda:0") for p in plan.parts], LoopbackComm(), CFG).solve()
    assert res.bounds == whole.bounds
    assert res.stop_reason == whole.stop_reason
    assert scatter_duals(plan, res.lam_parts, inst.flat.num_layers).tobytes() == whole.state.lam.tobytes()
