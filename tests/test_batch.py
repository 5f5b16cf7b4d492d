"""Batches of independent instances solved as one merged instance (config
C5; paper_2310_08230_b200/batch.py).

* CPU: the merged flat table is the block-diagonal union, and the oracle's
  averaging-only solve of it reproduces every instance's own solve bit for
  bit (the merge logic, independent of the GPU);
* GPU: the same for the product kernels (exact and deferred schedules,
  per-instance duals and bounds), and hybrid merged solves converge to every
  instance's own converged bound within 1e-5 relative.
"""

import numpy as np
import pytest

from paper_2310_08230_b200.batch import merge_instances
from paper_2310_08230_b200.config import SolveConfig


def _small_batch(n=3):
    from paper_2310_08230_b200 import product_space as ps
    from paper_2310_08230_b200.ilp import IlpInstance

    out = []
    for seed in range(n):
        M, N, fm, fn = ps.synthetic_pair("tetra" if seed % 2 else "icosa", seed)
        p = ps.build_product_space(M, N, fm, fn)
        out.append(IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, 128))
    return out


def _oracle(inst):
    from oracle import model

    f = inst.flat
    return model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts,
                                 {k: getattr(f, k) for k in ("bdd_layer_lo", "layer_node_lo", "layer_var",
                                                             "layer_bdd", "zero_t", "one_t", "proc_ptr",
                                                             "proc_layers")})


def test_merged_table_is_block_diagonal():
    insts = _small_batch()
    merged, idx = merge_instances(insts)
    f = merged.flat
    assert f.num_bdds == sum(i.flat.num_bdds for i in insts)
    for k, inst in enumerate(insts):
        g = inst.flat
        lo, hi = idx.layer[k], idx.layer[k + 1]
        assert np.array_equal(f.layer_var[lo:hi] - idx.var[k], g.layer_var)
        nlo, nhi = idx.node[k], idx.node[k + 1]
        z = f.zero_t[nlo:nhi]
        assert np.array_equal(np.where(z >= 0, z - nlo, z), g.zero_t)
        assert np.all((f.zero_t[nlo:nhi] < 0) | ((f.zero_t[nlo:nhi] >= nlo) & (f.zero_t[nlo:nhi] < nhi)))
    assert np.array_equal(np.sort(merged.variable_order), np.arange(merged.num_variables))


@pytest.mark.parametrize("schedule", ["exact", "deferred"])
def test_oracle_merged_averaging_equals_separate_solves(schedule):
    from oracle import solver

    insts = _small_batch()
    merged, idx = merge_instances(insts)
    oi, of = _oracle(merged)
    st, _, _ = solver.solve(oi, mode="mma-only", max_iterations=6, dual_tolerance=-np.inf, flat=of,
                            schedule=schedule)
    for k, inst in enumerate(insts):
        si, sf = _oracle(inst)
        s1, rec, _ = solver.solve(si, mode="mma-only", max_iterations=6, dual_tolerance=-np.inf, flat=sf,
                                  schedule=schedule)
        assert st.lam[idx.layer[k]:idx.layer[k + 1]].tobytes() == s1.lam.tobytes()
        assert float(np.sum(st.bounds[idx.bdd[k]:idx.bdd[k + 1]])) == rec[-1][2]


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["exact", "deferred"])
def test_gpu_merged_averaging_equals_separate_solves(schedule):
    from bench import build_instance
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.batch import solve_merged

    insts = [build_instance("c3", s) for s in (0, 5, 9)]
    cfg = SolveConfig(mode="mma-only", max_iterations=5, dual_tolerance=-np.inf, mma_schedule=schedule)
    res = solve_merged(insts, cfg, device="cuda:0")
    for k, inst in enumerate(insts):
        one = qn.solve(inst, cfg, device="cuda:0")
        assert res.lam(k).tobytes() == one.state.lam.tobytes()
        assert res.bounds[k] == one.bounds[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["exact", "deferred"])
def test_gpu_merged_hybrid_converges_to_every_instance_bound(schedule):
    from bench import build_instance
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.batch import solve_merged

    insts = [build_instance("c3", s) for s in (1, 2, 3, 4)]
    cfg = SolveConfig(mode="hybrid", mma_schedule=schedule, max_iterations=3000)
    res = solve_merged(insts, cfg, device="cuda:0")
    for k, inst in enumerate(insts):
        one = qn.solve(inst, SolveConfig(mode="hybrid", max_iterations=1000), device="cuda:0")
        assert abs(res.bounds[k] - one.best_bound) <= 1e-5 * abs(one.best_bound), (k, res.bounds[k], one.best_bound)


@pytest.mark.gpu
@pytest.mark.parametrize("schedule,compact", [("exact", 0.5), ("deferred", 0.5), ("exact", 0.0)])
def test_gpu_batched_hybrid_equals_separate_solves(schedule, compact):
    """BatchedSolver: every instance's own hybrid solve on one merged instance —
    records, stopping and duals bit for bit against qn.solve of each; with
    compaction the live instances are re-merged as others stop (the five
    separate solves stop at different iterations, so the batch shrinks)."""
    from bench import build_instance
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.batch import BatchedSolver

    insts = [build_instance("c3", s) for s in (0, 1, 3, 7, 13)]
    cfg = SolveConfig(mode="hybrid", mma_schedule=schedule, max_iterations=60 if schedule == "exact" else 120)
    solver = BatchedSolver(insts, cfg, device="cuda:0", compact=compact)
    got = solver.solve()
    assert (solver.repacks > 0) == (compact > 0)
    for k, inst in enumerate(insts):
        one = qn.solve(inst, cfg, device="cuda:0")
        assert got[k].bounds == one.bounds, k
        assert [r.kind for r in got[k].records] == [r.kind for r in one.records], k
        assert got[k].stop_reason == one.stop_reason and got[k].iterations == one.iterations
        assert got[k].best_bound == one.best_bound
        assert got[k].lam.tobytes() == one.state.lam.tobytes(), k


def test_batched_solver_runs_hybrid_solves_only():
    from paper_2310_08230_b200.batch import BatchedSolver

    with pytest.raises(ValueError, match="hybrid"):
        BatchedSolver([], SolveConfig(mode="mma-only"))


@pytest.mark.gpu
def test_gpu_batched_single_instance_equals_its_solve():
    """A batch of one: one batched iteration, then the instance's own
    DualSolver loop (the hand-off) — identical to qn.solve."""
    from bench import build_instance
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.batch import solve_batched

    inst = build_instance("c3", 1)
    cfg = SolveConfig(mode="hybrid", max_iterations=40)
    (got,) = solve_batched([inst], cfg, device="cuda:0")
    one = qn.solve(inst, cfg, device="cuda:0")
    assert got.bounds == one.bounds
    assert got.iterations == one.iterations and got.stop_reason == one.stop_reason
    assert got.lam.tobytes() == one.state.lam.tobytes()


@pytest.mark.gpu
def test_gpu_batched_time_limit_stops_every_instance():
    """max_seconds = 0: every instance stops after its first iteration with
    the time-limit reason, as its separate solve does."""
    from bench import build_instance
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.batch import solve_batched

    insts = [build_instance("c3", s) for s in (2, 4)]
    cfg = SolveConfig(mode="hybrid", max_iterations=30, max_seconds=0.0)
    got = solve_batched(insts, cfg, device="cuda:0")
    for g, inst in zip(got, insts):
        one = qn.solve(inst, cfg, device="cuda:0")
        assert g.stop_reason == one.stop_reason == "max_seconds"
        assert g.bounds == one.bounds and g.iterations == one.iterations == 1
