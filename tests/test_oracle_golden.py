"""Pin the CPU oracle (oracle/) against outputs of the real reference.

tests/golden/golden.json was produced by tests/golden/make_golden.py running
prodmatch itself; the oracle must reproduce every FlatBdds array, every
intermediate vector and the mma-only bound trajectory bit-for-bit, and the
hybrid trajectory within the OpenBLAS ddot tolerance.
"""

import numpy as np
import pytest

from oracle import model, solver
from tests.golden_util import FLAT_FIELDS, case_inputs, h, load_cases

CASES = load_cases()


def oracle_instance(case):
    costs, rows, chunk = case_inputs(case)
    if not isinstance(rows, list):
        rows = rows.rows()
    inst = model.instance_from_rows(costs, rows)
    if chunk:
        inst = model.split_instance(inst, chunk)
    return inst


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(case):
    inst = oracle_instance(case)
    flat = model.flatten(inst)
    for k in FLAT_FIELDS:
        assert h(getattr(flat, k)) == case["flat"][k], k
    assert h(inst.order) == case["flat"]["variable_order"]
    assert h(inst.costs) == case["flat"]["costs"]

    st = solver.init_duals(inst, flat)
    assert st.bound == case["init"]["bound"]
    assert h(st.lam) == case["init"]["lam"]
    st.mma(True)
    g = case["after_forward"]
    assert (st.bound, h(st.lam), h(st.F)) == (g["bound"], g["lam"], g["F"])
    m0, m1 = st.min_marginals()
    assert (h(m0), h(m1), h(st.B)) == (g["m0"], g["m1"], g["B"])
    st.mma(False)
    g = case["after_backward"]
    assert (st.bound, h(st.lam), h(st.B)) == (g["bound"], g["lam"], g["B"])
    assert h(st.subgradient()) == g["subgradient"]
    agrees, score, pref = solver.agreement_scores(st)
    assert (h(agrees), h(score), h(pref)) == tuple(case["agreement"][k] for k in ("agrees", "score", "preferred"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_solve_trajectories(case):
    inst = oracle_instance(case)
    g = case["mma-only"]
    st, rec, stop = solver.solve(inst, mode="mma-only", max_iterations=len(g["bounds"]) - 1 if g["stop"] == "max_iterations" else 10_000)
    assert [r[2] for r in rec] == g["bounds"]
    assert [r[1] for r in rec] == g["kinds"]
    assert stop == g["stop"] and h(st.lam) == g["lam"]
    g = case["hybrid"]
    st, rec, stop = solver.solve(inst, mode="hybrid", max_iterations=len(g["bounds"]) - 1 if g["stop"] == "max_iterations" else 10_000, dot="blas")
    got = np.array([r[2] for r in rec])
    ref = np.array(g["bounds"])
    n = min(len(got), len(ref))
    # OpenBLAS ddot order depends on the host; bounds agree to ~1e-12 relative
    assert np.allclose(got[:n], ref[:n], rtol=1e-9, atol=1e-9)
