"""Perturbation-based primal rounding (rounding.py, dm_perturb_round).

* GPU == oracle restatement (oracle/solver.py perturb_round + the exact
  averaging passes) round by round: disagreement counts and the final
  assignment bit for bit, same seed;
* the rounded assignment satisfies every constraint (every diagram accepts
  it; verify_solution on the product-space rows) and its gap is reported
  against the unperturbed bound; C4 is certified in seconds.
* CPU: the lock-step diagram walk (diagrams_accept) == Bdd.accepts.
"""

import numpy as np
import pytest

from paper_2310_08230_b200.rounding import diagrams_accept
from tests.golden_util import case_inputs, load_cases

CASES = {c["name"]: c for c in load_cases()}


def _inst(name):
    from paper_2310_08230_b200.ilp import IlpInstance, make_row

    costs, rows, chunk = case_inputs(CASES[name])
    if isinstance(rows, list):
        return IlpInstance.from_rows(costs, [make_row(*r) for r in rows], chunk_size=chunk)
    return IlpInstance.from_csr(rows.costs, rows.row_ptr, rows.row_var, rows.row_coef, rows.row_rhs, chunk)


@pytest.mark.parametrize("name", ["random1_c0", "random4_c3", "ps_tetra"])
def test_diagrams_accept_matches_bdd_accepts(name):
    inst = _inst(name)
    rng = np.random.default_rng(3)
    for _ in range(30):
        x = rng.integers(0, 2, inst.num_variables).astype(np.int8)
        got = diagrams_accept(inst.flat, x)
        want = [b.accepts(x[b.variables]) for b in inst.constraints]
        assert got.tolist() == want


def _oracle_rounding(inst, res_lam, seed, delta0, growth, per_round, max_rounds, boost=10.0):
    from oracle import model, solver

    f = inst.flat
    oi, of = model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts,
                                   {k: getattr(f, k) for k in ("bdd_layer_lo", "layer_node_lo", "layer_var",
                                                               "layer_bdd", "zero_t", "one_t", "proc_ptr",
                                                               "proc_layers")})
    st = solver.OracleDual(oi, of)
    st.set_lambda(res_lam)
    hist = []
    for r in range(max_rounds):
        values, _, dis = solver.perturb_round(st, delta0 * growth ** r, seed, r, boost)
        hist.append(dis)
        if dis == 0:
            return hist, values
        for _ in range(per_round):
            st.mma(True)
            st.mma(False)
    return hist, None


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ps_tetra", "ps_icosa", "ps_c1", "ps_c3"])
def test_gpu_rounding_matches_oracle_and_is_feasible(name):
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.rounding import perturbation_rounding

    inst = _inst(name)
    res = qn.solve(inst, SolveConfig(max_iterations=8))
    lam = res.state.lam
    delta0 = 1e-3 * float(np.median(np.abs(inst.costs[inst.costs != 0])))
    out = perturbation_rounding(res.state, seed=7, max_rounds=60, iterations_per_round=3, delta0=delta0, growth=1.2)
    hist, values = _oracle_rounding(inst, lam, 7, delta0, 1.2, 3, 60)
    assert out.disagree_history == hist
    assert out.assignment is not None and values is not None
    constrained = inst.constraint_counts > 0
    assert out.assignment[constrained].tobytes() == values[constrained].tobytes()
    assert diagrams_accept(inst.flat, out.assignment).all()
    assert out.objective >= res.best_bound - 1e-9 * abs(res.best_bound)


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["exact", "deferred"])
def test_gpu_rounding_certifies_c4_in_seconds(schedule):
    from bench import build_instance
    from paper_2310_08230_b200 import product_space as ps
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.rounding import perturbation_rounding

    inst = build_instance("c4", 0)
    res = qn.solve(inst, SolveConfig(mma_schedule=schedule, max_iterations=400))
    out = perturbation_rounding(res.state)
    assert out.status in ("certified", "feasible")
    assert out.seconds < 10.0
    p = ps.synthetic_product_space("c4", 0)
    assert not ps.verify_solution(p, out.assignment[: p.num_variables])
    assert out.report.primal_dual_gap < 1e-2
