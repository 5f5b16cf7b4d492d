"""B200 path == reference, through the C-ABI library (pytest -m gpu).

* every golden case (real-reference outputs): init duals, each exact pass,
  min-marginal table, subgradient, agreement scores and the mma-only
  trajectory bit-for-bit; hybrid trajectories bit-for-bit against the
  oracle in chunked-dot mode and within 1e-9 of the reference's BLAS run;
* kernel-level checks on random duals against the C oracle;
* numpy-order reductions, L-BFGS pieces and projection.
"""

import numpy as np
import pytest
import torch

from oracle import model, solver
from paper_2310_08230_b200 import qn
from paper_2310_08230_b200.config import SolveConfig
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, dual_objective, init_duals, mma_pass, subgradient
from paper_2310_08230_b200.errors import EmptyHistory
from paper_2310_08230_b200.ilp import IlpInstance, make_row
from paper_2310_08230_b200.kernels import dev_dot, dev_sum
from paper_2310_08230_b200.primal import agreement_scores
from tests.golden_util import case_inputs, h, load_cases

pytestmark = pytest.mark.gpu
CASES = load_cases()


def product_instance(case):
    costs, rows, chunk = case_inputs(case)
    if isinstance(rows, list):
        return IlpInstance.from_rows(costs, [make_row(*r) for r in rows], chunk_size=chunk)
    return IlpInstance.from_csr(rows.costs, rows.row_ptr, rows.row_var, rows.row_coef, rows.row_rhs, chunk)


def oracle_twin(inst):
    f = inst.flat
    arrays = {k: getattr(f, k) for k in ("bdd_layer_lo", "layer_node_lo", "layer_var", "layer_bdd", "zero_t",
                                          "one_t", "proc_ptr", "proc_layers")}
    return model.from_flat_table(inst.costs, inst.variable_order, f.constraint_counts, arrays)


MMA_KERNELS = {"node_parallel": 0, "per_copy": 1 << 18}  # dm_flat_set_mma_config lookahead-word bit 18


@pytest.mark.parametrize("kernels", list(MMA_KERNELS))
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_exact_passes_match_reference(case, kernels):
    inst = product_instance(case)
    st = init_duals(inst)
    st.dev.set_mma_config(256, 2, 0, False, (1 << 16) | MMA_KERNELS[kernels])
    assert st.bound == case["init"]["bound"]
    assert h(st.lam) == case["init"]["lam"]
    mma_pass(st, FORWARD)
    g = case["after_forward"]
    assert st.bound == g["bound"]
    assert h(st.lam) == g["lam"]
    assert h(st.F.cpu().numpy()) == g["F"]
    m0, m1 = st.min_marginal_table()
    assert (h(m0), h(m1)) == (g["m0"], g["m1"])
    assert h(st.B.cpu().numpy()) == g["B"]
    mma_pass(st, BACKWARD)
    g = case["after_backward"]
    assert (st.bound, h(st.lam), h(st.B.cpu().numpy())) == (g["bound"], g["lam"], g["B"])
    assert h(subgradient(st)) == g["subgradient"]
    sc = agreement_scores(st)
    assert (h(sc.agrees), h(sc.score), h(sc.preferred)) == tuple(
        case["agreement"][k] for k in ("agrees", "score", "preferred"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_argmin_from_backward_pass_decisions(case):
    inst = product_instance(case)
    st = init_duals(inst)
    for _ in range(2):
        mma_pass(st, FORWARD)
        mma_pass(st, BACKWARD)
        walk = torch.empty(st.flat.num_layers, dtype=torch.float64, device=st.device)
        st.dev.k_argmin(st.lam_d, st.B, walk)
        if st.dev.records_decisions:
            rec = torch.empty_like(walk)
            st.dev.k_argmin_from_pass(st.B, rec)
            assert rec.cpu().numpy().tobytes() == walk.cpu().numpy().tobytes()
        assert subgradient(st).tobytes() == walk.cpu().numpy().tobytes()
    with pytest.raises(ValueError):  # a table no backward pass wrote
        st.dev.k_argmin_from_pass(st.F, torch.empty_like(st.lam_d))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_mma_only_solve_matches_reference(case):
    inst = product_instance(case)
    g = case["mma-only"]
    iters = len(g["bounds"]) - 1 if g["stop"] == "max_iterations" else 10_000
    res = qn.solve(inst, SolveConfig(mode="mma-only", max_iterations=iters))
    assert res.bounds == g["bounds"]
    assert [r.kind for r in res.records] == g["kinds"]
    assert res.stop_reason == g["stop"]
    assert h(res.state.lam) == g["lam"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_hybrid_solve_matches_oracle_and_reference(case):
    inst = product_instance(case)
    g = case["hybrid"]
    iters = len(g["bounds"]) - 1 if g["stop"] == "max_iterations" else 10_000
    res = qn.solve(inst, SolveConfig(mode="hybrid", max_iterations=iters))
    oi, of = oracle_twin(inst)
    ost, orec, ostop = solver.solve(oi, mode="hybrid", max_iterations=iters, dot="chunked", flat=of)
    assert res.bounds == [r[2] for r in orec]  # bitwise, same reduction order
    assert [r.kind for r in res.records] == [r[1] for r in orec]
    assert res.stop_reason == ostop
    assert res.state.lam.tobytes() == ost.lam.tobytes()
    ref = np.array(g["bounds"])
    got = np.array(res.bounds)
    n = min(len(ref), len(got))
    assert np.allclose(got[:n], ref[:n], rtol=1e-9, atol=1e-9)  # OpenBLAS ddot order


@pytest.mark.parametrize("name", ["random3_c3", "random7_c0", "ps_tetra", "ps_icosa", "ps_c1"])
def test_sweep_kernels_on_random_duals(name):
    case = next(c for c in CASES if c["name"] == name)
    inst = product_instance(case)
    oi, of = oracle_twin(inst)
    rng = np.random.default_rng(1)
    for trial in range(3):
        lam = rng.standard_normal(of.num_layers) * (10.0 ** trial)
        ost = solver.OracleDual(oi, of)
        ost.lam[:] = lam
        ost.refresh_backward()
        ost.refresh_forward()
        st = init_duals(inst)
        st.set_lambda(lam)
        assert st.B.cpu().numpy().tobytes() == ost.B.tobytes()
        st.refresh_forward()
        assert st.F.cpu().numpy().tobytes() == ost.F.tobytes()
        assert st.bound == ost.bound
        m0, m1 = st.min_marginal_table()
        om0, om1 = ost.min_marginals()
        assert m0.tobytes() == om0.tobytes() and m1.tobytes() == om1.tobytes()
        assert subgradient(st).tobytes() == ost.subgradient().tobytes()
        d = rng.standard_normal(of.num_layers)
        dd = torch.as_tensor(d, device=st.device)
        for gamma in (0.0, 0.37, 3.1):
            assert st.eval_step(dd, gamma) == ost.eval_trial(d, gamma)
        # exact passes from arbitrary duals
        mma_pass(st, FORWARD)
        ost.mma(True)
        assert st.lam.tobytes() == ost.lam.tobytes() and st.bound == ost.bound
        mma_pass(st, BACKWARD)
        ost.mma(False)
        assert st.lam.tobytes() == ost.lam.tobytes() and st.bound == ost.bound


# 3849..4095 (and totals counts in that range) are the lengths whose numpy
# pairwise tree has 33 leaves
@pytest.mark.parametrize("n", [0, 1, 5, 7, 8, 9, 15, 16, 17, 127, 128, 129, 255, 256, 1000, 3849, 4095, 4096, 4097,
                               2 * 4096 + 4000, 65537, 636_800, 2_000_003, 3849 * 4096 - 7,
                               # more than 4096 chunks: totals reduced through the dm_sum tree
                               4096 * 4096, 4096 * 4096 + 1, 20_000_003, 40_000_000])
def test_pairwise_sum_and_dot_match_numpy(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 8, n)
    b = rng.standard_normal(n)
    ta, tb = torch.as_tensor(a, device="cuda"), torch.as_tensor(b, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    dev_sum(ta, out[0:1])
    dev_dot(ta, tb, out[1:2])
    got = out.cpu().numpy()
    assert got[0].tobytes() == np.sum(a).tobytes()
    assert got[1].tobytes() == np.float64(solver._dot_chunked(a, b)).tobytes()


def kinked():
    return IlpInstance.from_rows(np.array([4.0, 1.0, 3.0]), [make_row([0, 1], [1, 1], 1), make_row([0, 2], [1, 1], 1)])


def test_project_direction_reference_example():  # reference test_qn.py:40-44
    st = init_duals(kinked())
    d = qn.project_direction(np.array([3.0, 7.0, 1.0, -2.0]), st)
    assert d.tolist() == [1.0, 0.0, -1.0, 0.0]


def test_lbfgs_direction_requires_history():
    with pytest.raises(EmptyHistory):
        qn.lbfgs_direction(np.zeros(3), qn.LbfgsHistory(5))


def test_lbfgs_direction_matches_dense_oracle_and_pairwise_oracle():  # test_qn.py:62-75
    rng = np.random.default_rng(42)
    n = 12
    history = qn.LbfgsHistory(10)
    cfg = qn.StepConfig()
    pairs = []
    while len(history) < 7:
        s = rng.standard_normal(n)
        y = rng.standard_normal(n)
        if s @ y >= cfg.curvature_eps:
            qn.update_history(s, y, history, cfg)
            sy = solver._dot_chunked(s, y)
            pairs.insert(0, (s, y, 1.0 / sy, sy))
            pairs = pairs[:10]
        g = rng.standard_normal(n)
        d = qn.lbfgs_direction(g, history)
        ps = list(history.newest_first())
        s0, y0, _ = ps[0]
        s0, y0 = s0.cpu().numpy(), y0.cpu().numpy()
        H = np.eye(n) * (s0 @ y0) / (y0 @ y0)
        for s, y, rho in reversed(ps):
            s, y = s.cpu().numpy(), y.cpu().numpy()
            V = np.eye(n) - rho * np.outer(s, y)
            H = V @ H @ V.T + rho * np.outer(s, s)
        ref = H @ g
        assert np.abs(d - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max())
        assert d.tobytes() == solver.lbfgs(g, pairs, solver._dot_chunked).tobytes()


# up to ~590 chunks the recursion is one cooperative launch; 3,000,000 (733
# chunks) takes the per-step launches on a B200
@pytest.mark.parametrize("n,m", [(1, 1), (4096, 1), (3 * 4096 + 123, 4), (100003, 10), (4095, 3), (5 * 4096 + 3900, 5),
                                 (3_000_000, 3)])
def test_fused_two_loop_matches_unfused_and_oracle(n, m):
    rng = np.random.default_rng(n + m)
    history = qn.LbfgsHistory(10)
    pairs = []
    while len(history) < m:
        s = rng.standard_normal(n)
        y = s * rng.uniform(0.5, 2.0, n) + 0.01 * rng.standard_normal(n)
        sy = solver._dot_chunked(s, y)
        if sy >= 1e-8:
            qn.update_history(s, y, history, qn.StepConfig())
            pairs.insert(0, (s, y, 1.0 / sy, sy))
    g = torch.from_numpy(rng.standard_normal(n)).cuda()
    fused = qn.lbfgs_direction(g, history).cpu().numpy()
    plain = qn.lbfgs_direction(g, history, fused=False).cpu().numpy()
    assert fused.tobytes() == plain.tobytes()
    assert fused.tobytes() == solver.lbfgs(g.cpu().numpy(), pairs, solver._dot_chunked).tobytes()


def test_fused_two_loop_on_a_misaligned_gradient():
    """g as a view one element into its buffer: no 16-byte vector path, every
    chunk through the generic per-element path, same bits."""
    n, m = 3 * 4096 + 5, 2
    rng = np.random.default_rng(7)
    history = qn.LbfgsHistory(10)
    pairs = []
    while len(history) < m:
        s = rng.standard_normal(n)
        y = s * rng.uniform(0.5, 2.0, n)
        sy = solver._dot_chunked(s, y)
        qn.update_history(s, y, history, qn.StepConfig())
        pairs.insert(0, (s, y, 1.0 / sy, sy))
    big = torch.from_numpy(rng.standard_normal(n + 1)).cuda()
    g = big[1:]
    assert g.data_ptr() % 16 != 0
    fused = qn.lbfgs_direction(g, history).cpu().numpy()
    assert fused.tobytes() == solver.lbfgs(g.cpu().numpy(), pairs, solver._dot_chunked).tobytes()


def test_history_pool_reuses_evicted_pairs():
    h = qn.LbfgsHistory(3)
    like = torch.zeros(5, dtype=torch.float64, device="cuda")
    h.preallocate(like)
    seen = set()
    for k in range(8):
        s, y = h.reserve(like)
        seen.update((id(s), id(y)))
        s.fill_(k + 1.0)
        y.fill_(2.0 * (k + 1))
        if k != 4:  # one rejected pair: its storage stays in the pool
            h.push(s, y, 1.0, 1.0)
    assert len(seen) == 8  # memory + 1 pairs, never more
    assert [float(s[0]) for s, _, _ in h.newest_first()] == [8.0, 7.0, 6.0]
    assert [float(y[0]) for _, y, _ in h.newest_first()] == [16.0, 14.0, 12.0]


def test_find_step_size_kinked():  # test_qn.py:104-114
    st = init_duals(kinked())
    assert dual_objective(st) == pytest.approx(3.0)
    g = subgradient(st)
    assert g.tolist() == [0.0, 1.0, 1.0, 0.0]
    d = qn.project_direction(g, st)
    gamma, improved = qn.find_step_size(st, d, 1.0, qn.StepConfig(min_ascent=1e-3))
    assert improved
    assert st.eval_lambda(st.lam + gamma * d) == pytest.approx(3.5)


def test_find_step_size_counts():  # test_qn.py:117-137
    st = init_duals(kinked())
    calls = []
    orig = st.eval_step
    st.eval_step = lambda d, gm: (calls.append(1), orig(d, gm))[1]
    cfg = qn.StepConfig(min_ascent=1e-3, max_trials=5)
    gamma, improved = qn.find_step_size(st, np.zeros(4), 1.0, cfg, on_device=False)
    assert not improved and len(calls) == 6
    s0 = st.sweeps
    assert qn.find_step_size(st, np.zeros(4), 1.0, cfg) == (gamma, improved)
    assert st.sweeps - s0 == 6  # baseline plus K trials, on the device
    calls.clear()
    d = qn.project_direction(subgradient(st), st)
    cfg = qn.StepConfig(min_ascent=-10.0)
    host = qn.find_step_size(st, d, 1.0, cfg, on_device=False)
    assert len(calls) == 2
    s0 = st.sweeps
    assert qn.find_step_size(st, d, 1.0, cfg) == host
    assert st.sweeps - s0 == 2


@pytest.mark.parametrize("name", ["ps_tetra", "ps_icosa", "random3_c3", "random7_c0", "kinked"])
def test_device_step_search_matches_host_loop(name):
    """dm_step_search == the host trial loop (qn.py:132-159): same gamma, same
    verdict, same number of trial sweeps, over random directions, starting
    steps and ascent thresholds (incl. early stops and all-trials runs)."""
    inst = product_instance(next(c for c in CASES if c["name"] == name))
    st = init_duals(inst)
    mma_pass(st, FORWARD)
    mma_pass(st, BACKWARD)
    rng = np.random.default_rng(7)
    for trial in range(12):
        d = qn.project_direction(rng.standard_normal(st.lam.shape) * 10.0 ** rng.uniform(-4, 0), st)
        d = torch.from_numpy(np.asarray(d)).to(st.device)
        gamma0 = float(10.0 ** rng.uniform(-2, 1))
        cfg = qn.StepConfig(min_ascent=float([0.0, 1e-9, 1e-3, 1.0, -1.0][trial % 5]),
                            max_trials=int(rng.integers(1, 8)))
        s0 = st.sweeps
        host = qn.find_step_size(st, d, gamma0, cfg, on_device=False)
        n_host = st.sweeps - s0
        s0 = st.sweeps
        dev = qn.find_step_size(st, d, gamma0, cfg)
        assert dev == host
        assert st.sweeps - s0 == n_host


def test_solver_iteration_empty_history_is_averaging():  # test_qn.py:140-146
    st = init_duals(kinked())
    gamma, used = qn.solver_iteration(st, qn.LbfgsHistory(5), 1.0, qn.StepConfig())
    assert not used and gamma == 1.0
    assert dual_objective(st) == pytest.approx(4.0)


def test_free_variables_clamped():  # test_dual.py:84-90
    inst = IlpInstance.from_rows(np.array([-2.0, 1.0, 3.0]), [make_row([1], [1], 1)])
    st = init_duals(inst)
    assert st.free_values == {0: 1, 2: 0}
    assert dual_objective(st) == pytest.approx(-1.0)
    sums = st.lambda_sums()
    assert sums.tolist() == [-2.0, 1.0, 3.0]
    sc = agreement_scores(st)
    assert not sc.agrees[0] and not sc.agrees[2]


def _wide_dense_rows(seed, n_vars, n_rows, row_len, coef_max, hub_vars):
    """Random feasible equality rows: coefficients 1..coef_max (layer widths grow
    with the number of distinct partial sums); every row also contains the
    `hub_vars`, so those variables have n_rows copies."""
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(n_rows):
        vs = rng.choice(np.arange(hub_vars, n_vars), size=row_len - hub_vars, replace=False)
        vs = np.concatenate([np.arange(hub_vars), vs]).astype(np.int64)
        cs = rng.integers(1, coef_max + 1, size=len(vs)).astype(np.int64)
        pick = rng.random(len(vs)) < 0.5
        rows.append((vs, cs, int(cs[pick].sum())))
    return rng.standard_normal(n_vars), rows


@pytest.mark.parametrize("seed,row_len,coef_max,n_rows,hubs", [
    (0, 12, 4, 6, 0),    # layers wider than 8: per-copy W=16 / W=32 kernels
    (1, 14, 6, 6, 0),
    (2, 6, 1, 12, 2),    # variables with 12 copies: per-copy K=32 kernels
    (3, 12, 5, 12, 2),   # both
])
def test_exact_passes_wide_and_dense_instances(seed, row_len, coef_max, n_rows, hubs):
    costs, rows = _wide_dense_rows(seed, 40, n_rows, row_len, coef_max, hubs)
    inst = IlpInstance.from_rows(costs, [make_row(*r) for r in rows])
    f = inst.flat
    assert f.max_width > 8 or f.max_degree > 8
    oi, of = oracle_twin(inst)
    ost = solver.init_duals(oi, of)
    st = init_duals(inst)
    assert st.lam.tobytes() == ost.lam.tobytes() and st.bound == ost.bound
    for _ in range(3):
        mma_pass(st, FORWARD)
        ost.mma(True)
        assert st.lam.tobytes() == ost.lam.tobytes() and st.bound == ost.bound
        assert st.F.cpu().numpy().tobytes() == ost.F.tobytes()
        mma_pass(st, BACKWARD)
        ost.mma(False)
        assert st.lam.tobytes() == ost.lam.tobytes() and st.bound == ost.bound
        assert st.B.cpu().numpy().tobytes() == ost.B.tobytes()
        assert subgradient(st).tobytes() == ost.subgradient().tobytes()


def test_solve_batch_matches_sequential_solves():
    insts = [product_instance(c) for c in CASES if c["name"] in ("ps_tetra", "ps_icosa", "random3_c3", "random7_c0")]
    cfg = SolveConfig(mode="hybrid", max_iterations=8)
    seq = [qn.solve(i, cfg) for i in insts]
    for k in (2, 3):
        bat = qn.solve_batch(insts, cfg, concurrency=k)
        for a, b in zip(seq, bat):
            assert a.bounds == b.bounds
            assert a.state.lam.tobytes() == b.state.lam.tobytes()


@pytest.mark.parametrize("n", [1, 7, 4095, 4096, 4097, 3 * 4096 + 5, 100003])
def test_curvature_pair_matches_separate_ops(n):
    from paper_2310_08230_b200.kernels import dev_curvature_pair

    rng = np.random.default_rng(n)
    lam, lp, g, gp = (torch.from_numpy(rng.standard_normal(n)).cuda() for _ in range(4))
    s, y = torch.empty_like(lam), torch.empty_like(lam)
    sy = torch.empty(1, dtype=torch.float64, device=lam.device)
    lp_before = lp.clone()
    dev_curvature_pair(lam, lp, g, gp, s, y, sy)
    s_ref = lam.cpu().numpy() - lp_before.cpu().numpy()
    y_ref = gp.cpu().numpy() - g.cpu().numpy()
    assert s.cpu().numpy().tobytes() == s_ref.tobytes()
    assert y.cpu().numpy().tobytes() == y_ref.tobytes()
    assert lp.cpu().numpy().tobytes() == lam.cpu().numpy().tobytes()
    assert float(sy[0]) == solver._dot_chunked(s_ref, y_ref)


def _host_level_order(f, forward):
    """build_mma_schedule (dm_host.cpp) restated: level = 1 + deepest level of
    the copies' previous (forward) / next (backward) layers; positions with
    copies bucketed by level in visitation order."""
    pp, pl, bl, lb = (np.asarray(getattr(f, k)) for k in ("proc_ptr", "proc_layers", "bdd_layer_lo", "layer_bdd"))
    P = len(pp) - 1
    last = np.zeros(len(bl) - 1, np.int64)
    lev = np.full(P, -1, np.int64)
    ks = range(P) if forward else range(P - 1, -1, -1)
    for p in ks:
        ls = pl[pp[p]:pp[p + 1]]
        if len(ls) == 0:
            continue
        js = lb[ls]
        first = ls == bl[js] if forward else ls + 1 == bl[js + 1]
        v = int((last[js[~first]] + 1).max()) if (~first).any() else 0
        last[js] = v
        lev[p] = v
    visit = np.fromiter(ks, np.int64)
    visit = visit[lev[visit] >= 0]
    order = visit[np.argsort(lev[visit], kind="stable")]
    return order, lev[order]


@pytest.mark.parametrize("name", ["ps_tetra", "ps_icosa", "ps_c1", "random3_c3", "random7_c0", "toy"])
def test_device_level_orders_match_host_schedule(name):
    from paper_2310_08230_b200 import _native

    inst = product_instance(next(c for c in CASES if c["name"] == name))
    st = init_duals(inst)
    f = inst.flat
    pp, pl = np.asarray(f.proc_ptr), np.asarray(f.proc_layers)
    for forward in (True, False):
        order, lev = _host_level_order(f, forward)
        n = st.dev.info["fw_tasks" if forward else "bw_tasks"]
        assert n == len(order)
        assert st.dev.info["fw_depth" if forward else "bw_depth"] == (int(lev.max()) + 1 if len(lev) else 0)
        levels = np.zeros(n, np.int32)
        layers = np.zeros(n * 8, np.int32)
        _native.check(_native.load().dm_flat_task_levels(st.dev.handle, int(forward), levels.ctypes.data,
                                                        layers.ctypes.data))
        assert levels.tolist() == lev.tolist()
        want = np.full((n, 8), -1, np.int64)
        for t, p in enumerate(order):
            k = pp[p + 1] - pp[p]
            want[t, :k] = pl[pp[p]:pp[p + 1]]
        assert layers.reshape(n, 8).tolist() == want.tolist()


@pytest.mark.parametrize("where", ["inner_true", "skip_layer", "last_to_node", "bad_code"])
def test_invalid_arc_targets_are_rejected(where):
    import copy

    from paper_2310_08230_b200.errors import ProdmatchError
    from paper_2310_08230_b200.kernels import DeviceFlat

    inst = product_instance(next(c for c in CASES if c["name"] == "random3_c0"))
    t = copy.copy(inst.flat)
    t.zero_t, t.one_t = t.zero_t.copy(), t.one_t.copy()
    bl, lnl = t.bdd_layer_lo, t.layer_node_lo
    j = int(np.argmax(np.diff(bl) >= 3))  # a diagram with at least three layers
    l0 = int(bl[j])
    if where == "inner_true":
        t.zero_t[lnl[l0]] = -2
    elif where == "skip_layer":
        t.one_t[lnl[l0]] = lnl[l0 + 2]
    elif where == "last_to_node":
        t.zero_t[lnl[bl[j + 1] - 1]] = 0
    else:
        t.one_t[lnl[l0]] = -3
    DeviceFlat(inst.flat, torch.device("cuda:0"))  # the untouched table is accepted
    with pytest.raises(ProdmatchError, match="arc targets"):
        DeviceFlat(t, torch.device("cuda:0"))


@pytest.mark.parametrize("k", range(1, 9))
def test_exact_pass_division_matches_ddiv(k):
    """The exact passes divide a copy-delta sum by the copy count with a
    prepared reciprocal (+ Markstein's correction for 3, 5, 6, 7): bit-equal
    to IEEE division on 2^26 hashed doubles per count."""
    import ctypes

    from paper_2310_08230_b200 import _native

    bad = ctypes.c_ulonglong(0)
    _native.check(_native.load().dm_debug_div_check(k, 1 << 26, 12345 + k, ctypes.byref(bad)))
    assert bad.value == 0


@pytest.mark.parametrize("n", [4096 * 4096 + 4096, 20_000_003, 40_000_001])
def test_two_loop_and_curvature_pair_beyond_4096_chunks(n):
    """The fused L-BFGS two-loop and the curvature pair on vectors longer than
    4096 chunks, bitwise against the oracle's two-loop in chunked-dot order."""
    from paper_2310_08230_b200.kernels import dev_curvature_pair, dev_lbfgs_direction

    rng = np.random.default_rng(5)
    dev = torch.device("cuda")
    pairs_h, pairs_d = [], []
    for _ in range(3):
        s_ = rng.standard_normal(n)
        y_ = s_ + 0.1 * rng.standard_normal(n)
        sy = solver._dot_chunked(s_, y_)
        pairs_h.append((s_, y_, 1.0 / sy, sy))
        pairs_d.append((torch.as_tensor(s_, device=dev), torch.as_tensor(y_, device=dev), 1.0 / sy, sy))
    g = rng.standard_normal(n)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    dev_lbfgs_direction(torch.as_tensor(g, device=dev), pairs_d, d)
    want = solver.lbfgs(g, pairs_h, solver._dot_chunked)
    assert d.cpu().numpy().tobytes() == want.tobytes()
    lam, lam_prev = torch.as_tensor(rng.standard_normal(n), device=dev), torch.as_tensor(rng.standard_normal(n), device=dev)
    gg, gp = torch.as_tensor(rng.standard_normal(n), device=dev), torch.as_tensor(rng.standard_normal(n), device=dev)
    s_o, y_o = torch.empty_like(lam), torch.empty_like(lam)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    want_sy = solver._dot_chunked((lam - lam_prev).cpu().numpy(), (gp - gg).cpu().numpy())
    dev_curvature_pair(lam, lam_prev, gg, gp, s_o, y_o, out)
    assert float(out.item()) == want_sy


def test_layers_wider_than_32_raise_unsupported_instance():
    """dm_flat_create's envelope: a cardinality row whose
    diagram has a 33-node layer raises the typed error, not a crash."""
    from paper_2310_08230_b200.errors import UnsupportedInstance

    n = 70
    inst = IlpInstance.from_rows(np.arange(n, dtype=np.float64), [make_row(list(range(n)), [1] * n, 32)],
                                 chunk_size=0)
    assert inst.flat.max_width >= 33
    with pytest.raises(UnsupportedInstance):
        init_duals(inst)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_solve_on_a_non_current_device_restores_the_current_device():
    inst = kinked()
    torch.cuda.set_device(0)
    res = qn.solve(inst, SolveConfig(max_iterations=3), device="cuda:1")
    assert torch.cuda.current_device() == 0
    assert res.state.device == torch.device("cuda", 1)


def test_release_caches_then_reductions_still_match():
    """dm_release_caches frees the cached plans / scratch; later reductions
    rebuild them and still give numpy's bits."""
    from paper_2310_08230_b200.kernels import release_caches

    rng = np.random.default_rng(11)
    a = rng.standard_normal(100_003)
    ta = torch.as_tensor(a, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    dev_sum(ta, out[0:1])
    dev_dot(ta, ta, out[1:2])
    release_caches()
    dev_sum(ta, out[0:1])
    dev_dot(ta, ta, out[1:2])
    got = out.cpu().numpy()
    assert got[0].tobytes() == np.sum(a).tobytes()
    assert got[1].tobytes() == np.float64(solver._dot_chunked(a, a)).tobytes()
