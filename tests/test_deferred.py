"""The deferred (throughput) averaging schedule — SolveConfig(mma_schedule="deferred").

There is no reference implementation of it (the reference runs the
sequential passes, kernels.py:162-362; the paper's GPU solver uses FastDOG's
parallel deferred averaging), so parity is two-level:

* bit for bit against its C restatement (oracle/ckernels.c oracle_dfr_*,
  oracle/solver.py OracleDual.deferred_round): every pass output (duals,
  distance tables, escrow, averages, bounds) and whole solves in both modes;
* at convergence against the exact schedule (whose duals are the
  reference's, tests/test_gpu_parity.py): the same converged dual bound
  within 1e-5 relative (north star's tolerance) on C1, C3 and C4.

CPU tests check the restatement's own invariants (dual feasibility after a
round, monotone bounds, bound <= brute-force optimum).
"""

import os

import numpy as np
import pytest
import torch

from oracle import model, solver
from tests.golden_util import FLAT_FIELDS, case_inputs, load_cases

CASES = load_cases()
SMALL = [c for c in CASES if c["name"] in ("random0_c0", "random3_c3", "random7_c0", "kinked", "toy", "ps_tetra",
                                           "ps_icosa", "ps_c1", "ps_c3")]


def oracle_instance(case):
    costs, rows, chunk = case_inputs(case)
    if not isinstance(rows, list):
        rows = rows.rows()
    inst = model.instance_from_rows(costs, rows)
    if chunk:
        inst = model.split_instance(inst, chunk)
    return inst, model.flatten(inst)


def _brute_force_optimum(costs, rows):
    import itertools

    n = len(costs)
    best = np.inf
    for bits in itertools.product((0, 1), repeat=n):
        x = np.array(bits)
        if all(int(np.dot(c, x[v])) == b for v, c, b in rows):
            best = min(best, float(np.dot(costs, x)))
    return best


@pytest.mark.parametrize("seed", range(10))
def test_oracle_deferred_round_invariants(seed):
    case = next(c for c in CASES if c["name"] == f"random{seed}_c0")
    costs, rows, _ = case_inputs(case)
    inst, flat = oracle_instance(case)
    st = solver.init_duals(inst, flat)
    opt = _brute_force_optimum(costs, rows)
    prev = st.objective()
    for _ in range(6):
        st.deferred_round(0.5)
        b = st.objective()
        assert b >= prev - 1e-9 * max(1.0, abs(prev))  # monotone
        assert b <= opt + 1e-9 * max(1.0, abs(opt))  # a lower bound
        sums = st.lambda_sums()
        assert np.allclose(sums, inst.costs, rtol=1e-12, atol=1e-12)  # feasible after the flush
        prev = b


def test_oracle_deferred_converges_to_exact_bound_icosa():
    case = next(c for c in CASES if c["name"] == "ps_icosa")
    inst, flat = oracle_instance(case)
    _, rec_e, _ = solver.solve(inst, mode="hybrid", max_iterations=200, dot="chunked", flat=flat)
    _, rec_d, _ = solver.solve(inst, mode="hybrid", max_iterations=200, dot="chunked", flat=flat,
                               schedule="deferred", damping=0.5)
    be, bd = max(r[2] for r in rec_e), max(r[2] for r in rec_d)
    assert abs(be - bd) <= 1e-5 * abs(be)


# --------------------------------------------------------------------------- GPU
def gpu_instance(case):
    from paper_2310_08230_b200.ilp import IlpInstance, make_row

    costs, rows, chunk = case_inputs(case)
    if isinstance(rows, list):
        return IlpInstance.from_rows(costs, [make_row(*r) for r in rows], chunk_size=chunk)
    return IlpInstance.from_csr(rows.costs, rows.row_ptr, rows.row_var, rows.row_coef, rows.row_rhs, chunk)


def oracle_twin(inst):
    f = inst.flat
    return model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts,
                                 {k: getattr(f, k) for k in FLAT_FIELDS})


def _nodes(st, x_il):
    import torch

    out = torch.empty(st.flat.num_nodes, dtype=torch.float64, device=st.device)
    st.dev.dfr_to_nodes(x_il, out)
    return out.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["node_parallel", "interleaved"])
@pytest.mark.parametrize("omega", [0.5, 0.3])
@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_deferred_passes_match_oracle(case, omega, layout, monkeypatch):
    """Each pass of a round, from arbitrary duals, bit for bit — both kernel
    families: node-parallel on node-order tables (dm_dfr_np_*) and lane per
    diagram on the interleaved sweep layout (dm_dfr_*)."""
    from oracle.clib import lib, ptr
    from paper_2310_08230_b200.dual import init_duals

    monkeypatch.setenv("DM_DFR_NP", "0" if layout == "interleaved" else "1")
    inst = gpu_instance(case)
    oi, of = oracle_twin(inst)
    rng = np.random.default_rng(7)
    lam = rng.standard_normal(of.num_layers) * 3.0
    st = init_duals(inst, schedule="deferred")
    if layout == "node_parallel" and not st._np:
        pytest.skip("instance outside the node-parallel passes' envelope")
    if st._np:
        F_t, B_t, fw, bw = st.F, st.B, st.dev.dfr_np_forward, st.dev.dfr_np_backward
        nodes = lambda x: x.cpu().numpy()  # noqa: E731
    else:
        F_t, B_t, fw, bw = st.F_il, st.B_il, st.dev.dfr_forward, st.dev.dfr_backward
        nodes = lambda x: _nodes(st, x)  # noqa: E731
    st.set_lambda(lam)  # refresh_backward: B and its decisions
    ost = solver.OracleDual(oi, of)
    ost.lam[:] = lam
    ost.refresh_backward()
    assert nodes(B_t).tobytes() == ost.B.tobytes()
    assert st.bound == ost.bound
    geo = (of.num_bdds, ptr(of.bdd_layer_lo), ptr(of.layer_node_lo), ptr(of.zero_t), ptr(of.one_t))
    P = len(of.proc_ptr) - 1
    mbar, avg, bounds = np.zeros(of.num_layers), np.zeros(of.num_layers), np.zeros(of.num_bdds)
    # forward pass
    fw(omega, st.lam_d, None, B_t, F_t, st.mbar, st._bounds)
    lib.oracle_dfr_forward(*geo, omega, ptr(ost.lam), None, ptr(ost.B), ptr(ost.F), ptr(mbar), ptr(bounds))
    assert st.lam.tobytes() == ost.lam.tobytes()
    assert nodes(F_t).tobytes() == ost.F.tobytes()
    assert st.mbar.cpu().numpy().tobytes() == mbar.tobytes()
    assert st._bounds.cpu().numpy().tobytes() == bounds.tobytes()
    # average
    st.dev.dfr_average(st.mbar, st.avg)
    lib.oracle_dfr_average(P, ptr(of.proc_ptr), ptr(of.proc_layers), ptr(mbar), ptr(avg))
    assert st.avg.cpu().numpy().tobytes() == avg.tobytes()
    # backward pass (adds the forward escrow)
    bw(omega, st.lam_d, st.avg, F_t, B_t, st.mbar, st._bounds)
    lib.oracle_dfr_backward(*geo, omega, ptr(ost.lam), ptr(avg), ptr(ost.F), ptr(ost.B), ptr(mbar), ptr(bounds))
    assert st.lam.tobytes() == ost.lam.tobytes()
    assert nodes(B_t).tobytes() == ost.B.tobytes()
    assert st.mbar.cpu().numpy().tobytes() == mbar.tobytes()
    assert st._bounds.cpu().numpy().tobytes() == bounds.tobytes()
    # flush: average + a sweep adding it == dm_dfr_flush (average into lam) + a plain sweep
    lam2, B2, b2 = st.lam_d.clone(), B_t.clone(), st._bounds.clone()
    st.dev.dfr_average(st.mbar, st.avg)
    bw(0.0, lam2, st.avg, None, B2, None, b2)
    st.dev.dfr_flush(st.mbar, st.lam_d)
    bw(0.0, st.lam_d, None, None, B_t, None, st._bounds, True)
    lib.oracle_dfr_average(P, ptr(of.proc_ptr), ptr(of.proc_layers), ptr(mbar), ptr(avg))
    lib.oracle_dfr_backward(*geo, 0.0, ptr(ost.lam), ptr(avg), None, ptr(ost.B), None, ptr(bounds))
    for lam_t, Bx, b_t in ((st.lam_d, B_t, st._bounds), (lam2, B2, b2)):
        assert lam_t.cpu().numpy().tobytes() == ost.lam.tobytes()
        assert nodes(Bx).tobytes() == ost.B.tobytes()
        assert b_t.cpu().numpy().tobytes() == bounds.tobytes()
    # the recorded decisions walk to the full argmin
    bits = torch.empty(of.num_layers, dtype=torch.float64, device=st.device)
    st.dev.k_argmin_from_pass(B_t, bits)
    assert bits.cpu().numpy().tobytes() == ost.subgradient().tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["node_parallel", "interleaved"])
@pytest.mark.parametrize("mode", ["mma-only", "hybrid"])
@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_deferred_solve_matches_oracle(case, mode, layout, monkeypatch):
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig
    from paper_2310_08230_b200.dual import subgradient
    from paper_2310_08230_b200.primal import agreement_scores

    monkeypatch.setenv("DM_DFR_NP", "0" if layout == "interleaved" else "1")
    inst = gpu_instance(case)
    oi, of = oracle_twin(inst)
    iters = 12
    res = qn.solve(inst, SolveConfig(mode=mode, max_iterations=iters, mma_schedule="deferred", mma_damping=0.4))
    ost, orec, ostop = solver.solve(oi, mode=mode, max_iterations=iters, dot="chunked", flat=of,
                                    schedule="deferred", damping=0.4)
    assert res.bounds == [r[2] for r in orec]
    assert [r.kind for r in res.records] == [r[1] for r in orec]
    assert res.stop_reason == ostop
    assert res.state.lam.tobytes() == ost.lam.tobytes()
    # consumers of the interleaved tables: decision walk, min-marginals, agreement
    assert subgradient(res.state).tobytes() == ost.subgradient().tobytes()
    m0, m1 = res.state.min_marginal_table()
    om0, om1 = ost.min_marginals()
    assert m0.tobytes() == om0.tobytes() and m1.tobytes() == om1.tobytes()
    sc = agreement_scores(res.state)
    oa, os_, op = solver.agreement_scores(ost)
    assert (sc.agrees.tobytes(), sc.score.tobytes()) == (oa.tobytes(), os_.tobytes())


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["c1", "c3", "c4"])
def test_deferred_converges_to_the_exact_bound(cfg):
    """Converged dual bound of the deferred schedule == the exact schedule's
    (the reference's) within 1e-5 relative."""
    from bench import build_instance
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig

    inst = build_instance(cfg, 0)
    ex = qn.solve(inst, SolveConfig(mode="hybrid", max_iterations=400))
    df = qn.solve(inst, SolveConfig(mode="hybrid", max_iterations=2000, mma_schedule="deferred"))
    assert abs(ex.best_bound - df.best_bound) <= 1e-5 * abs(ex.best_bound), (ex.best_bound, df.best_bound)
    b = df.bounds
    assert all(b1 >= b0 - 1e-9 * max(1.0, abs(b0)) for b0, b1 in zip(b, b[1:]))  # monotone up to rounding


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_deferred_full_size_matches_oracle(cfg):
    """Two hybrid iterations of the deferred schedule at the benched sizes,
    bit for bit against the oracle (chunked-dot order)."""
    from bench import build_instance
    from paper_2310_08230_b200 import qn
    from paper_2310_08230_b200.config import SolveConfig

    inst = build_instance(cfg, 0)
    oi, of = oracle_twin(inst)
    res = qn.solve(inst, SolveConfig(mode="hybrid", max_iterations=3, mma_schedule="deferred"))
    ost, orec, _ = solver.solve(oi, mode="hybrid", max_iterations=3, dot="chunked", flat=of, schedule="deferred",
                                threads=os.cpu_count())
    assert res.bounds == [r[2] for r in orec]
    assert res.state.lam.tobytes() == ost.lam.tobytes()
