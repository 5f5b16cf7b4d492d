"""Primal recovery against the reference's own outputs (tests/golden/primal.json,
made by tests/golden/make_primal_golden.py running prodmatch.primal).

CPU part: the native conditioning (dm_condition_flat) applied to the fixes
the oracle's agreement scores choose must rebuild the reference's residual
instance array for array.  GPU part: fix_and_reduce and recover_primal on
the device duals of the same mma-only solve.
"""

import math

import numpy as np
import pytest

from oracle import model, solver
from paper_2310_08230_b200 import primal
from paper_2310_08230_b200.errors import EmptyFeasibleSet
from paper_2310_08230_b200.ilp import IlpInstance, make_row
from tests.golden_util import FLAT_FIELDS, case_inputs, h, load_primal_cases

CASES = load_primal_cases()


def instances(case):
    costs, rows, chunk = case_inputs(case)
    if isinstance(rows, list):
        ours = IlpInstance.from_rows(costs, [make_row(*r) for r in rows], chunk_size=chunk)
        orows = rows
    else:
        ours = IlpInstance.from_csr(rows.costs, rows.row_ptr, rows.row_var, rows.row_coef, rows.row_rhs, chunk)
        orows = rows.rows()
    oi = model.instance_from_rows(costs, orows)
    if chunk:
        oi = model.split_instance(oi, chunk)
    return ours, oi


def chosen_fixes(agrees, score, preferred, fraction):
    agreeing = np.flatnonzero(agrees)
    take = int(math.floor(fraction * len(agreeing) + 1e-9))
    order = np.lexsort((agreeing, -score[agreeing]))
    return {int(v): int(preferred[v]) for v in agreeing[order[:take]]}


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_conditioning_rebuilds_reference_residual(case):
    ours, oi = instances(case)
    ost, _, _ = solver.solve(oi, mode="mma-only", max_iterations=case["mma_iterations"], dual_tolerance=0.0)
    assert ost.best_bound == case["best_bound"]
    agrees, score, preferred = solver.agreement_scores(ost)
    for frac, g in case["fix"].items():
        values = chosen_fixes(agrees, score, preferred, float(frac))
        if g.get("infeasible"):
            with pytest.raises(EmptyFeasibleSet):
                primal.condition_instance(ours, values)
            continue
        keys = sorted(values)
        assert h(np.array(keys, np.int64)) == g["fixed_vars"]
        assert h(np.array([values[k] for k in keys], np.int64)) == g["fixed_vals"]
        residual, dropped = primal.condition_instance(ours, values)
        assert residual.num_constraints == g["num_constraints"]
        assert dropped == g["dropped"]
        for k in FLAT_FIELDS:
            assert h(getattr(residual.flat, k)) == g["flat"][k], (frac, k)


def test_conditioning_keeps_untouched_and_rejects_contradictions():
    # x0 + x1 == 1 and x1 + x2 == 1
    inst = IlpInstance.from_rows(np.array([1.0, 2.0, 3.0]), [make_row([0, 1], [1, 1], 1), make_row([1, 2], [1, 1], 1)])
    same, dropped = primal.condition_instance(inst, {})
    assert dropped == 0 and same.num_constraints == 2
    for k in FLAT_FIELDS:
        assert h(getattr(same.flat, k)) == h(getattr(inst.flat, k))
    res, dropped = primal.condition_instance(inst, {1: 1})  # forces x0 = x2 = 0: both rows become chains
    assert dropped == 0 or res.num_constraints == 2 - dropped
    with pytest.raises(EmptyFeasibleSet):
        primal.condition_instance(inst, {0: 1, 1: 1})


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_recover_primal_matches_reference(case):
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig

    ours, _ = instances(case)
    res = qn.solve(ours, SolveConfig(mode="mma-only", max_iterations=case["mma_iterations"], dual_tolerance=0.0))
    st = res.state
    assert st.best_bound == case["best_bound"]
    for frac, g in case["fix"].items():
        if g.get("infeasible"):
            with pytest.raises(primal.InfeasibleAfterFixing):
                primal.fix_and_reduce(ours, st, float(frac))
            continue
        partial, residual = primal.fix_and_reduce(ours, st, float(frac))
        assert len(partial) == g["num_fixed"]
        for k in FLAT_FIELDS:
            assert h(getattr(residual.flat, k)) == g["flat"][k], (frac, k)
    if "recover" not in case:  # fix-only case (reference B&B hit its time budget)
        return
    sol = primal.recover_primal(ours, st, SolveConfig(max_seconds=60.0))
    want = case["recover"]
    assert sol.status == want["status"]
    assert sol.ladder_stage == want["ladder_stage"]
    if "objective" in want:
        assert float(ours.costs @ sol.assignment) == pytest.approx(want["objective"], rel=1e-12, abs=1e-12)
        assert h(np.asarray(sol.assignment, np.int8)) == want["assignment"]
