"""Parity at the BENCHED sizes: bench.py's C2 line (320 x 320 full product
space, 31 M nodes), the north star's C4 target (980 x 980 k-NN pruned pair)
and two members of the C5 batch (C3-generator seeds 17 and 42).

``tests/golden/golden_large.json`` holds the REAL reference's outputs on
these instances (``tests/golden/make_golden.py --large`` ran ``prodmatch``
here: C2's build alone takes 91 s): the FlatBdds hashes, the bound and
duals after initialisation and after each exact pass, the min-marginal
table, the subgradient, the agreement scores, and 3 mma-only + 3 hybrid
iterations.  Checked here:

* CPU: the native lowering reproduces every FlatBdds array bit for bit;
* GPU: the exact passes, min-marginals, subgradient, agreement scores and
  the mma-only trajectory bit for bit against the reference's hashes;
* GPU: the hybrid trajectory bit for bit against the C oracle (chunked-dot
  order; it runs these sizes in seconds per iteration) and within 1e-9 of
  the reference's OpenBLAS run.
"""

import json
import os

import numpy as np
import pytest

from tests.golden_util import FLAT_FIELDS, h

GOLDEN_LARGE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_large.json")
with open(GOLDEN_LARGE) as fh:
    CASES = json.load(fh)["cases"]
IDS = [c["name"] for c in CASES]

_cache: dict = {}


def instance(case):
    """The lowered instance of a large case (built once per process)."""
    from paper_2310_08230_b200.ilp import IlpInstance
    from tests.cases import csr_hash, product_space

    key = case["name"]
    if key not in _cache:
        p = product_space(case["config"], case.get("seed", 0))
        assert csr_hash(p) == case["rows_hash"], "product-space builder output changed"
        _cache.clear()  # one large instance resident at a time
        _cache[key] = IlpInstance.from_csr(p.costs, p.row_ptr, p.row_var, p.row_coef, p.row_rhs, case["chunk"])
    return _cache[key]


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_large_lowering_matches_reference(case):
    inst = instance(case)
    f = inst.flat
    assert {"variables": inst.num_variables, "bdds": f.num_bdds, "layers": f.num_layers,
            "nodes": f.num_nodes} == case["sizes"]
    for k in FLAT_FIELDS:
        assert h(getattr(f, k)) == case["flat"][k], k
    assert h(inst.variable_order) == case["flat"]["variable_order"]
    assert h(inst.costs) == case["flat"]["costs"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_large_exact_passes_match_reference(case):
    from paper_2310_08230_b200.dual import BACKWARD, FORWARD, init_duals, mma_pass, subgradient
    from paper_2310_08230_b200.primal import agreement_scores

    st = init_duals(instance(case))
    assert st.bound == case["init"]["bound"]
    assert h(st.lam) == case["init"]["lam"]
    mma_pass(st, FORWARD)
    g = case["after_forward"]
    assert (st.bound, h(st.lam), h(st.F.cpu().numpy())) == (g["bound"], g["lam"], g["F"])
    m0, m1 = st.min_marginal_table()
    assert (h(m0), h(m1), h(st.B.cpu().numpy())) == (g["m0"], g["m1"], g["B"])
    mma_pass(st, BACKWARD)
    g = case["after_backward"]
    assert (st.bound, h(st.lam), h(st.B.cpu().numpy())) == (g["bound"], g["lam"], g["B"])
    assert h(subgradient(st)) == g["subgradient"]
    sc = agreement_scores(st)
    assert (h(sc.agrees), h(sc.score), h(sc.preferred)) == tuple(
        case["agreement"][k] for k in ("agrees", "score", "preferred"))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_large_mma_only_solve_matches_reference(case):
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig

    g = case["mma-only"]
    res = qn.solve(instance(case), SolveConfig(mode="mma-only", max_iterations=len(g["bounds"]) - 1))
    assert res.bounds == g["bounds"]
    assert [r.kind for r in res.records] == g["kinds"]
    assert h(res.state.lam) == g["lam"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_large_hybrid_solve_matches_oracle_and_reference(case):
    from oracle import model, solver
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig

    inst = instance(case)
    g = case["hybrid"]
    iters = len(g["bounds"]) - 1
    res = qn.solve(inst, SolveConfig(mode="hybrid", max_iterations=iters))
    f = inst.flat
    oi, of = model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts,
                                   {k: getattr(f, k) for k in FLAT_FIELDS})
    ost, orec, ostop = solver.solve(oi, mode="hybrid", max_iterations=iters, dot="chunked", flat=of,
                                    threads=os.cpu_count())
    assert res.bounds == [r[2] for r in orec]  # bitwise, same reduction order
    assert [r.kind for r in res.records] == [r[1] for r in orec] == g["kinds"]
    assert res.state.lam.tobytes() == ost.lam.tobytes()
    assert np.allclose(res.bounds, g["bounds"], rtol=1e-9, atol=1e-9)  # OpenBLAS ddot order
