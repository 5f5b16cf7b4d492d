"""The reference's behavioural unit tests, restated against the B200 path
(pytest -m gpu). Each test names the reference test it mirrors
(/root/reference/pkg/tests/test_dual.py, test_qn.py, test_primal.py); the
expected values are the reference's, and where the reference freezes them
with its brute-force oracle (tests/bruteforce.py) this file carries its own
enumerator (`ilp_optimum`, `accepted_min`) that never touches the diagram
code under test.
"""

import numpy as np
import pytest
import torch

from paper_2310_08230_b200 import qn
from paper_2310_08230_b200.config import SolveConfig
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, dual_objective, init_duals, mma_pass, subgradient
from paper_2310_08230_b200.errors import EmptyFeasibleSet
from paper_2310_08230_b200.ilp import IlpInstance, make_row
from paper_2310_08230_b200.primal import (INFEASIBLE, OPTIMAL, TIMEOUT, PartialAssignment, agreement_scores,
                                          exact_solve, fix_and_reduce, make_gap_report, recover_primal)

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- helpers

def ilp_optimum(costs, rows):
    """(value, x) of the cheapest 0-1 vector meeting every equality row, by
    enumerating all 2^n vectors; None when infeasible. Ties: first in
    big-endian order."""
    costs = np.asarray(costs, np.float64)
    n = len(costs)
    x = ((np.arange(1 << n)[:, None] >> np.arange(n - 1, -1, -1)[None, :]) & 1).astype(np.int64)
    ok = np.ones(len(x), bool)
    for v, c, b in rows:
        ok &= x[:, np.asarray(v)] @ np.asarray(c) == b
    if not ok.any():
        return None
    vals = x[ok] @ costs
    k = int(np.argmin(vals))
    return float(vals[k]), x[ok][k]


def rows_of(inst):
    return [(r.variables, r.coefficients, r.rhs) for r in inst.rows]


def accepted_min(bdd, lam):
    """min over the diagram's accepted vectors of lam . x, plus per-layer
    (m0, m1) min-marginals, by enumeration."""
    sols = np.array(list(bdd.enumerate_accepted()), np.float64)
    vals = sols @ lam
    m0 = [vals[sols[:, i] == 0].min(initial=np.inf) for i in range(sols.shape[1])]
    m1 = [vals[sols[:, i] == 1].min(initial=np.inf) for i in range(sols.shape[1])]
    return float(vals.min()), np.array(m0), np.array(m1)


def feasibility_residual(state):
    c = state.instance.costs
    return float(np.max(np.abs(state.lambda_sums() - c) / (1.0 + np.abs(c))))


def toy():
    return IlpInstance.from_rows(np.array([1.0, 1.0, 1.0]), [make_row([0, 1], [1, 1], 1), make_row([1, 2], [1, 1], 1)])


def kinked():
    # E(t) = min(t, 1) + min(4 - t, 3): strictly peaked at t == 1 with E == 4
    return IlpInstance.from_rows(np.array([4.0, 1.0, 3.0]), [make_row([0, 1], [1, 1], 1), make_row([0, 2], [1, 1], 1)])


def random_any_rhs(rng, num_vars, num_rows):
    """test_dual.py:93-111: rhs anywhere in the row's range (may be infeasible)."""
    rows = []
    tries = 0
    while len(rows) < num_rows and tries < 50 * num_rows:
        tries += 1
        k = int(rng.integers(2, min(6, num_vars) + 1))
        v = np.sort(rng.choice(num_vars, size=k, replace=False))
        c = rng.integers(-2, 3, size=k)
        if not c.any():
            continue
        rows.append(make_row(v, c, int(rng.integers(int(np.minimum(c, 0).sum()), int(np.maximum(c, 0).sum()) + 1))))
    try:
        return IlpInstance.from_rows(rng.standard_normal(num_vars) * 3.0, rows)
    except EmptyFeasibleSet:
        return None


def random_witnessed(rng, num_vars=10, num_rows=4, feasible=True):
    """test_primal.py:27-40: rhs from one shared witness, so jointly feasible."""
    w = rng.integers(0, 2, size=num_vars)
    rows = []
    for _ in range(num_rows):
        k = int(rng.integers(2, min(6, num_vars) + 1))
        v = np.sort(rng.choice(num_vars, size=k, replace=False))
        c = rng.integers(-2, 3, size=k)
        if not c.any():
            c[0] = 1
        local = w[v] if feasible else rng.integers(0, 2, size=k)
        rows.append(make_row(v, c, int(c @ local)))
    return IlpInstance.from_rows(rng.standard_normal(num_vars) * 2.0, rows)


def assert_feasible(inst, x):
    for bdd in inst.constraints:
        assert bdd.accepts([x[v] for v in bdd.variables])


# ---------------------------------------------------------------- dual (test_dual.py)

def test_init_duals_splits_costs_uniformly():  # test_dual.py:31-36
    st = init_duals(toy())
    assert st.lambda_of(0).tolist() == [1.0, 0.5]
    assert st.lambda_of(1).tolist() == [0.5, 1.0]
    assert dual_objective(st) == pytest.approx(1.0)
    assert feasibility_residual(st) < 1e-12


def test_zero_cost_instance_has_zero_dual():  # test_dual.py:39-42
    st = init_duals(IlpInstance.from_rows(np.zeros(3), [make_row([0, 1, 2], [1, 1, 1], 1)]))
    assert dual_objective(st) == 0.0


def test_variable_in_single_constraint_receives_full_cost():  # test_dual.py:45-48
    st = init_duals(IlpInstance.from_rows(np.array([3.0, 4.0]), [make_row([0, 1], [1, 1], 1)]))
    assert st.lambda_of(0).tolist() == [3.0, 4.0]


def test_mma_pass_keeps_toy_instance_at_its_optimum():  # test_dual.py:51-56
    st = init_duals(toy())
    mma_pass(st, FORWARD)
    mma_pass(st, BACKWARD)
    assert dual_objective(st) == pytest.approx(1.0)
    assert feasibility_residual(st) < 1e-12


def test_mma_is_noop_on_single_constraint_instances():  # test_dual.py:59-65
    st = init_duals(IlpInstance.from_rows(np.array([0.3, -1.5, 2.0]), [make_row([0, 1, 2], [1, 1, 1], 2)]))
    before = st.lam.copy()
    mma_pass(st, FORWARD)
    mma_pass(st, BACKWARD)
    assert np.allclose(st.lam, before, atol=1e-15)


def test_subgradient_toy_agreement_certificate():  # test_dual.py:68-74
    st = init_duals(toy())
    assert subgradient(st).tolist() == [0.0, 1.0, 1.0, 0.0]
    assert dual_objective(st) == pytest.approx(1.0)


def test_subgradient_forced_variable():  # test_dual.py:77-81
    st = init_duals(IlpInstance.from_rows(np.array([5.0, 0.2]), [make_row([0], [1], 1), make_row([0, 1], [1, 1], 1)]))
    assert subgradient(st)[0] == 1.0


@pytest.mark.parametrize("seed", range(8))
def test_passes_are_monotone_and_bounded_by_optimum(seed):  # test_dual.py:114-133
    inst = random_any_rhs(np.random.default_rng(seed), 10, 4)
    if inst is None:
        pytest.skip("degenerate draw")
    ref = ilp_optimum(inst.costs, rows_of(inst))
    st = init_duals(inst)
    values = [dual_objective(st)]
    for _ in range(25):
        mma_pass(st, FORWARD)
        values.append(dual_objective(st))
        mma_pass(st, BACKWARD)
        values.append(dual_objective(st))
        assert feasibility_residual(st) < 1e-9
    assert (np.diff(values) >= -1e-9).all()
    if ref is not None:
        assert values[-1] <= ref[0] + 1e-9


def test_min_marginal_table_matches_enumeration():  # test_dual.py:136-150
    inst = random_any_rhs(np.random.default_rng(3), 8, 3)
    st = init_duals(inst)
    mma_pass(st, FORWARD)
    m0, m1 = st.min_marginal_table()
    lo = inst.flat.bdd_layer_lo
    for j, bdd in enumerate(inst.constraints):
        _, e0, e1 = accepted_min(bdd, st.lambda_of(j))
        n = len(bdd.variables)
        np.testing.assert_allclose(m0[lo[j]:lo[j] + n], e0, rtol=0, atol=1e-12)
        np.testing.assert_allclose(m1[lo[j]:lo[j] + n], e1, rtol=0, atol=1e-12)


def test_kernel_bound_matches_enumerated_min_assignment():  # test_dual.py:153-160
    inst = random_any_rhs(np.random.default_rng(7), 9, 4)
    st = init_duals(inst)
    total = sum(accepted_min(b, st.lambda_of(j))[0] for j, b in enumerate(inst.constraints))
    assert dual_objective(st) == pytest.approx(total + st.free_contribution, abs=1e-12)


def test_results_identical_across_launch_shapes():  # test_dual.py:163-180 (thread counts -> launch shapes)
    inst = random_any_rhs(np.random.default_rng(11), 12, 5)
    outputs = []
    for threads, blocks, word in ((256, 3, 1 << 16), (128, 1, 1 << 16), (256, 2, (1 << 16) | (1 << 18)),
                                  (64, 4, 1 << 18)):
        st = init_duals(inst)
        st.dev.set_mma_config(threads, blocks, 0, False, word)
        for _ in range(5):
            mma_pass(st, FORWARD)
            mma_pass(st, BACKWARD)
        outputs.append((st.lam.copy(), dual_objective(st), subgradient(st)))
    for lam, obj, bits in outputs[1:]:
        assert lam.tobytes() == outputs[0][0].tobytes()
        assert obj == outputs[0][1]
        assert bits.tobytes() == outputs[0][2].tobytes()


@pytest.mark.parametrize("seed", [0, 1, 17, 256, 999, 4242, 7777, 10000])
def test_forced_variables_never_leak_infinities(seed):  # test_dual.py:183-202 (hypothesis seeds -> fixed seeds)
    rows = [([0], [1], 1), ([0, 1, 2], [1, 1, 1], 3), ([1, 2], [1, -1], 0)]
    costs = np.random.default_rng(seed).standard_normal(3) * 2.0
    st = init_duals(IlpInstance.from_rows(costs, [make_row(*r) for r in rows]))
    for _ in range(6):
        mma_pass(st, FORWARD)
        mma_pass(st, BACKWARD)
        assert np.isfinite(st.lam).all()
        assert feasibility_residual(st) < 1e-9
    assert dual_objective(st) <= ilp_optimum(costs, rows)[0] + 1e-9


# ---------------------------------------------------------------- qn (test_qn.py)

def test_project_direction_zero_sum_property():  # test_qn.py:47-54
    rng = np.random.default_rng(0)
    st = init_duals(kinked())
    for _ in range(25):
        d = qn.project_direction(rng.standard_normal(4), st)
        sums = np.zeros(3)
        np.add.at(sums, st.flat.layer_var, np.asarray(d))
        assert np.abs(sums).max() <= 1e-12


def test_lbfgs_direction_is_linear_in_g():  # test_qn.py:78-86
    h = qn.LbfgsHistory(4)
    qn.update_history(np.ones(5), np.arange(1.0, 6.0), h, qn.StepConfig())
    assert np.allclose(qn.lbfgs_direction(np.zeros(5), h), 0.0)
    g = np.random.default_rng(1).standard_normal(5)
    assert np.allclose(qn.lbfgs_direction(2.0 * g, h), 2.0 * qn.lbfgs_direction(g, h))


def test_update_history_curvature_gate_and_eviction():  # test_qn.py:89-101
    cfg = qn.StepConfig(curvature_eps=1e-8)
    h = qn.LbfgsHistory(3)
    s = np.array([1.0, 0.0])
    qn.update_history(s, np.array([0.0, 1.0]), h, cfg)  # s.y == 0: rejected
    assert len(h) == 0
    qn.update_history(s, np.array([1.0, 0.0]), h, cfg)
    assert len(h) == 1
    for k in range(4):
        qn.update_history(s * (k + 2), s, h, cfg)
    assert len(h) == 3
    assert float(h.newest()[0][0]) == 5.0  # the oldest pairs were evicted


def test_find_step_size_ascends_above_start():  # test_qn.py:104-114
    st = init_duals(kinked())
    d = qn.project_direction(subgradient(st), st)
    gamma, improved = qn.find_step_size(st, d, 1.0, qn.StepConfig(min_ascent=1e-3))
    assert improved
    d = np.asarray(d.cpu() if torch.is_tensor(d) else d)
    assert st.eval_lambda(st.lam + gamma * d) > dual_objective(st)


def test_find_step_size_breaks_once_ascent_threshold_met():  # test_qn.py:128-137
    """Any trial counts as sufficient ascent: the search stops after the
    baseline and one trial — on the host loop (its fused trial evaluations
    counted) and in the device search (its trial counter)."""
    st = init_duals(kinked())
    d = qn.project_direction(subgradient(st), st)
    cfg = qn.StepConfig(min_ascent=-10.0)
    calls = []
    original = st.eval_step
    st.eval_step = lambda dd, gamma: (calls.append(1), original(dd, gamma))[1]
    qn.find_step_size(st, d, 1.0, cfg, on_device=False)
    assert len(calls) == 2
    del st.eval_step
    _, _, trials = st.search_step(qn.as_device(d, st.device), 1.0, cfg.shrink, cfg.grow, cfg.min_ascent,
                                  cfg.max_trials)
    assert trials == 2


def test_lbfgs_direction_requires_history():  # test_qn.py:57-59
    from paper_2310_08230_b200.errors import EmptyHistory

    with pytest.raises(EmptyHistory):
        qn.lbfgs_direction(np.zeros(3), qn.LbfgsHistory(5))


def test_solver_iteration_keeps_optimal_toy_unchanged():  # test_qn.py:149-158
    st = init_duals(toy())
    before = dual_objective(st)
    h = qn.LbfgsHistory(5)
    for _ in range(3):
        qn.solver_iteration(st, h, 1.0, qn.StepConfig())
    assert dual_objective(st) == pytest.approx(before)


def test_solve_records_are_monotone_and_bounded():  # test_qn.py:161-182
    rng = np.random.default_rng(5)
    rows = []
    for _ in range(6):
        k = int(rng.integers(2, 6))
        v = np.sort(rng.choice(14, size=k, replace=False))
        c = rng.integers(-2, 3, size=k)
        if not c.any():
            continue
        rows.append(make_row(v, c, int(c @ rng.integers(0, 2, size=k))))
    inst = IlpInstance.from_rows(rng.standard_normal(14) * 2.0, rows)
    res = qn.solve(inst, SolveConfig(max_iterations=60))
    assert (np.diff(res.bounds) >= -1e-9).all()
    ref = ilp_optimum(inst.costs, rows_of(inst))
    if ref is not None:
        assert res.best_bound <= ref[0] + 1e-9
    assert res.records[0].kind == "init"
    assert res.records[1].kind == "mma"  # empty history on the first iteration


def test_mma_only_mode_never_takes_newton_steps():  # test_qn.py:185-188
    res = qn.solve(kinked(), SolveConfig(mode="mma-only", max_iterations=30))
    assert all(r.kind != "hybrid" for r in res.records)


# ---------------------------------------------------------------- primal (test_primal.py)

def test_agreement_votes_on_shared_variable():  # test_primal.py:43-50
    sc = agreement_scores(init_duals(toy()))
    assert sc.agrees.all()
    assert sc.preferred.tolist() == [0, 1, 0]
    assert sc.score[1] == pytest.approx(1.0)
    assert sc.score[0] == pytest.approx(0.5)


def test_agreement_disagreeing_variable():  # test_primal.py:53-61
    inst = IlpInstance.from_rows(np.array([0.0, 1.0, 1.0]), [make_row([0, 1], [1, 1], 1), make_row([1, 2], [1, 1], 1)])
    st = init_duals(inst)
    st.set_lambda(np.array([0.0, 1.0, 0.0, 1.0]))
    sc = agreement_scores(st)
    assert not sc.agrees[1]
    assert sc.agrees[0] and sc.preferred[0] == 1
    assert sc.agrees[2] and sc.preferred[2] == 0


def test_agreement_forced_variable_scores_infinite():  # test_primal.py:64-70
    sc = agreement_scores(init_duals(IlpInstance.from_rows(np.array([7.0]), [make_row([0], [1], 1)])))
    assert sc.agrees[0] and sc.preferred[0] == 1 and sc.score[0] == np.inf


def test_fix_all_with_full_agreement_empties_instance():  # test_primal.py:73-77
    partial, reduced = fix_and_reduce(toy(), init_duals(toy()), fraction=1.0)
    assert partial.values == {0: 0, 1: 1, 2: 0}
    assert reduced.num_constraints == 0


def test_fix_top_variable_collapses_constraints():  # test_primal.py:80-88
    inst = toy()
    partial, reduced = fix_and_reduce(inst, init_duals(inst), fraction=0.34)
    assert partial.values == {1: 1}
    assert reduced.num_constraints == 2
    for bdd in reduced.constraints:
        assert bdd.count_accepting_paths() == 1


def test_fixing_never_contradicts_a_single_constraint():  # test_primal.py:91-104
    rng = np.random.default_rng(2)
    for _ in range(20):
        inst = random_witnessed(rng)
        st = init_duals(inst)
        st.shift_lambda(qn.project_direction(rng.standard_normal(st.lam.shape), st))
        st.refresh_backward()
        partial, _ = fix_and_reduce(inst, st, fraction=1.0)
        partial.validate(inst)


def test_exact_solve_toy():  # test_primal.py:107-111
    res = exact_solve(toy())
    assert res.status == OPTIMAL
    assert res.assignment.tolist() == [0, 1, 0]
    assert res.objective == pytest.approx(1.0)


def test_exact_solve_detects_contradiction():  # test_primal.py:114-117
    inst = IlpInstance.from_rows(np.zeros(1), [make_row([0], [1], 0), make_row([0], [1], 1)])
    assert exact_solve(inst).status == INFEASIBLE


def test_exact_solve_matches_enumeration_on_random_instances():  # test_primal.py:120-137
    rng = np.random.default_rng(9)
    for _ in range(15):
        inst = random_witnessed(rng, num_vars=12, num_rows=5)
        ref = ilp_optimum(inst.costs, rows_of(inst))
        res = exact_solve(inst)
        assert ref is not None and res.status == OPTIMAL
        assert res.objective == pytest.approx(ref[0], abs=1e-9)
        assert_feasible(inst, res.assignment)


def test_exact_solve_respects_preassignment():  # test_primal.py:140-148
    inst = IlpInstance.from_rows(np.array([1.0, 2.0, 3.0]), [make_row([0, 1, 2], [1, 1, 1], 1)])
    res = exact_solve(inst, preassigned=PartialAssignment({0: 0, 1: 0}))
    assert res.status == OPTIMAL
    assert res.assignment.tolist() == [0, 0, 1]
    assert res.objective == pytest.approx(3.0)


def test_exact_solve_timeout():  # test_primal.py:151-156
    inst = IlpInstance.from_rows(np.linspace(0.0, 1.0, 14), [make_row(list(range(14)), [1] * 14, 7)])
    ticks = iter(np.arange(0.0, 5000.0, 0.5))
    assert exact_solve(inst, time_limit=1e-9, clock=lambda: next(ticks)).status == TIMEOUT


def test_gap_report_edges():  # test_primal.py:159-166
    rep = make_gap_report(10.0, 9.95)
    assert rep.primal_dual_gap == pytest.approx(0.005)
    assert rep.certified
    assert make_gap_report(0.0, 0.0).certified
    assert make_gap_report(0.0, -1e-12).certified
    assert not make_gap_report(0.0, -5.0).certified
    assert not make_gap_report(10.0, 8.0).certified


def test_recover_primal_toy_certified():  # test_primal.py:169-176
    inst = toy()
    rec = recover_primal(inst, qn.solve(inst, SolveConfig(max_iterations=30)).state)
    assert rec.status == "certified"
    assert rec.assignment.tolist() == [0, 1, 0]
    assert rec.report.primal_dual_gap == pytest.approx(0.0, abs=1e-9)
    assert rec.ladder_stage == 0


def test_recover_primal_ladder_backs_off_on_joint_infeasibility():  # test_primal.py:179-194
    inst = IlpInstance.from_rows(np.array([0.0, 1.0, 1.0]), [make_row([0, 1], [1, 1], 1), make_row([1, 2], [1, 1], 1)])
    st = init_duals(inst)
    st.set_lambda(np.array([0.0, 1.0, 0.0, 1.0]))
    rec = recover_primal(inst, st, SolveConfig(fixing_fraction=1.0))
    assert rec.status in ("feasible", "certified")
    assert rec.ladder_stage >= 1
    assert_feasible(inst, rec.assignment)


def test_recover_primal_random_suite_always_feasible():  # test_primal.py:197-218
    rng = np.random.default_rng(31)
    for _ in range(10):
        inst = random_witnessed(rng)
        ref = ilp_optimum(inst.costs, rows_of(inst))
        res = qn.solve(inst, SolveConfig(max_iterations=40))
        rec = recover_primal(inst, res.state)
        assert ref is not None and rec.assignment is not None
        x = rec.assignment
        assert_feasible(inst, x)
        assert float(inst.costs @ x) >= res.state.best_bound - 1e-9
        if rec.status == "certified":
            assert float(inst.costs @ x) == pytest.approx(ref[0], abs=1e-6)
