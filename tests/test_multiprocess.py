"""Multi-process path of bench.py on CPU (gloo, world_size 2).

Instance sharding (config C5 semantics): every rank solves its own product
space instance (seed = rank) with no collective on the data path; the only
collective is the report's (sum of work, max of time).  Here the per-rank
solve is the CPU oracle on a small product space, so the test checks the
sharding + aggregation logic without a GPU.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


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
        import time

        import bench
        from oracle import model, solver
        from tests.cases import product_case

        costs, rows, _ = product_case("tetra", seed=rank)
        inst = model.split_instance(model.instance_from_rows(costs, rows), 128)
        t0 = time.perf_counter()
        st, rec, _ = solver.solve(inst, mode="hybrid", max_iterations=5, threads=1)
        ms = (time.perf_counter() - t0) * 1e3
        work = st.sweeps * 2 * model.flatten(inst).num_nodes
        total, slowest = bench.aggregate_work_time(work, ms, world)
        out[rank] = (work, ms, total, slowest, rec[-1][2])
    finally:
        dist.destroy_process_group()


def test_instance_sharding_aggregation_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    works = [out[r][0] for r in range(world)]
    times = [out[r][1] for r in range(world)]
    for r in range(world):
        assert out[r][2] == pytest.approx(sum(works))
        assert out[r][3] == pytest.approx(max(times))
    # different seeds -> different instances -> different bounds
    assert out[0][4] != out[1][4]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c5_batch_shards_every_instance_once(world):
    import bench

    shares = [bench.c5_seeds(r, world) for r in range(world)]
    flat = sorted(s for sh in shares for s in sh)
    assert flat == list(range(bench.C5_INSTANCES))
    assert max(map(len, shares)) - min(map(len, shares)) <= 1
