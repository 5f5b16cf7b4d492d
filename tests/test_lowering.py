"""Native lowering (csrc/dm_host.cpp) == reference IlpInstance.from_rows ->
split_instance -> FlatBdds, bit-for-bit (golden hashes of the real reference)."""

import numpy as np
import pytest

from paper_2310_08230_b200 import product_space as ps
from paper_2310_08230_b200.ilp import IlpInstance, build_equality_bdd, make_row
from paper_2310_08230_b200.errors import EmptyFeasibleSet
from paper_2310_08230_b200.splitting import split_instance
from tests.golden_util import FLAT_FIELDS, case_inputs, h, load_cases

CASES = load_cases()


def product_instance(case):
    costs, rows, chunk = case_inputs(case)
    if isinstance(rows, list):
        inst = IlpInstance.from_rows(costs, [make_row(*r) for r in rows], chunk_size=chunk)
    else:
        inst = IlpInstance.from_csr(rows.costs, rows.row_ptr, rows.row_var, rows.row_coef, rows.row_rhs, chunk)
    return inst


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_native_lowering_matches_reference(case):
    inst = product_instance(case)
    f = inst.flat
    for k in FLAT_FIELDS:
        assert h(getattr(f, k)) == case["flat"][k], k
    assert h(inst.variable_order) == case["flat"]["variable_order"]
    assert h(inst.costs) == case["flat"]["costs"]


@pytest.mark.parametrize("case", [c for c in CASES if c["chunk"]], ids=lambda c: c["name"])
def test_split_instance_on_unsplit_instance(case):
    costs, rows, chunk = case_inputs(case)
    if isinstance(rows, list):
        base = IlpInstance.from_rows(costs, [make_row(*r) for r in rows])
    else:
        base = IlpInstance.from_csr(rows.costs, rows.row_ptr, rows.row_var, rows.row_coef, rows.row_rhs, 0)
    inst = split_instance(base, chunk)
    for k in FLAT_FIELDS:
        assert h(getattr(inst.flat, k)) == case["flat"][k], k


def test_cardinality_diagram_shape():  # reference test_bdd.py:19-23
    b = build_equality_bdd([1] * 8, 2, range(8))
    assert b.widths == [1, 2, 3, 3, 3, 3, 3, 2]
    assert b.count_accepting_paths() == 28


def test_infeasible_row_raises():
    with pytest.raises(EmptyFeasibleSet):
        build_equality_bdd([1, 1], 3, [0, 1])
    with pytest.raises(EmptyFeasibleSet):
        IlpInstance.from_rows(np.zeros(2), [make_row([0, 1], [2, 2], 1)])


def test_signed_pair():
    b = build_equality_bdd([1, -1], 0, [0, 1])
    assert sorted(b.enumerate_accepted()) == [(0, 0), (1, 1)]


def test_product_space_statistics():  # SPEC.md:408-412, acceptance 7
    for cfg, expect in (("tetra", 368), ("icosa", 8880)):
        M, N, fm, fn = ps.synthetic_pair(cfg)
        p = ps.build_product_space(M, N, fm, fn)
        assert p.num_variables == expect
        kinds = np.bincount(p.kind, minlength=5)
        if cfg == "tetra":
            assert kinds.tolist() == [48, 144, 16, 144, 16]
        assert 20 <= p.num_variables / (M.num_faces * N.num_faces) <= 24
        assert (p.costs >= 0).all()
        # every product triangle: 3 boundary incidences, <= 1 A^M and <= 1 A^N row
        nb = p.num_boundary_rows
        occ = np.bincount(p.row_var[: p.row_ptr[nb]], minlength=p.num_variables)
        assert (occ == 3).all()


def test_identity_matching_is_feasible():  # SPEC.md:440-446, acceptance 6
    M, N, fm, fn = ps.synthetic_pair("icosa")
    p = ps.build_product_space(M, N, fm, fm)
    # identity: tri-tri of every face with itself in the same rotation
    x = np.zeros(p.num_variables, np.int64)
    sel = (p.kind == ps.TRI_TRI) & (p.m == p.n).all(axis=1)
    x[sel] = 1
    assert sel.sum() == M.num_faces
    assert ps.verify_solution(p, x) == []
    assert abs(p.costs[sel].sum()) < 1e-12
    assert len(ps.verify_solution(p, np.zeros(p.num_variables, np.int64))) >= M.num_faces + N.num_faces
