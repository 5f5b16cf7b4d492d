"""Size-independent properties at BASELINE's full single-GPU workload (C2:
320×320-triangle product space, 2.29 M variables, 31 M BDD nodes), on the
GPU.  The oracle cannot run these sizes in seconds; instead:

* the two exact-pass kernel families (node-parallel and per-copy, built on
  different schedules) give bit-identical duals, distances and bounds;
* a pass is deterministic (repeated from the same state: same bits);
* dual feasibility (sum over copies == cost, test_dual.py:24-27) holds after
  the passes and a quasi-Newton step;
* the subgradient walked from the backward pass's recorded decisions equals
  the full argmin sweep, bit for bit;
* the device step search equals the host trial loop;
* bounds never decrease across exact passes (test_dual.py:114-133).

The same properties run on C4 (980 x 980 triangles, k-NN pruned, 3.5 M nodes).
"""

import numpy as np
import pytest
import torch

from paper_2310_08230_b200 import qn
from paper_2310_08230_b200.config import SolveConfig
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, dual_objective, init_duals, mma_pass, subgradient_device

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["c2", "c4"])
def c2(request):
    """The full single-GPU workloads: C2 (full product space) and C4 (the
    ~1000 x 1000-triangle k-NN pruned pair)."""
    from bench import build_instance

    return build_instance(request.param, 0)


def _feasibility(st):
    c = st.instance.costs
    return float(np.max(np.abs(st.lambda_sums() - c) / (1.0 + np.abs(c))))


def test_c2_kernel_families_agree_bitwise(c2):
    runs = []
    for word in ((1 << 16) | (1 << 18), (1 << 16)):  # per-copy (bit 18), then node-parallel (the default)
        st = init_duals(c2, device="cuda:0")
        st.dev.set_mma_config(256, 3, 32, False, word)
        bounds = [dual_objective(st)]
        for _ in range(2):
            mma_pass(st, FORWARD)
            bounds.append(dual_objective(st))
            mma_pass(st, BACKWARD)
            bounds.append(dual_objective(st))
        runs.append((st.lam.tobytes(), st.B.cpu().numpy().tobytes(), bounds))
        assert all(b1 >= b0 - 1e-9 * max(1.0, abs(b0)) for b0, b1 in zip(bounds, bounds[1:]))
    assert runs[0] == runs[1]


def test_c2_pass_determinism_feasibility_and_decisions(c2):
    st = init_duals(c2, device="cuda:0")
    assert _feasibility(st) < 1e-12
    mma_pass(st, FORWARD)
    mma_pass(st, BACKWARD)
    lam0, B0 = st.lam_d.clone(), st.B.clone()
    # the same backward pass again from the same state: the same bits
    mma_pass(st, FORWARD)
    mma_pass(st, BACKWARD)
    lam1, B1 = st.lam_d.clone(), st.B.clone()
    st.lam_d.copy_(lam0)
    st.B.copy_(B0)
    st.f_valid, st.b_valid = False, True
    mma_pass(st, FORWARD)
    mma_pass(st, BACKWARD)
    assert torch.equal(st.lam_d, lam1) and torch.equal(st.B, B1)
    assert _feasibility(st) < 1e-9
    # argmin from the pass's decisions == the full argmin sweep
    walk = subgradient_device(st).clone()
    full = torch.empty_like(walk)
    st.dev.k_argmin(st.lam_d, st.B, full)
    assert torch.equal(walk, full)


def test_c2_device_step_search_and_hybrid_iterations(c2):
    run = qn.DualSolver(c2, SolveConfig(mode="hybrid", max_iterations=10**9, dual_tolerance=0.0),
                        device="cuda:0").start()
    for _ in range(4):
        run.step()
    st = run.state
    g = subgradient_device(st)
    d = qn.project_direction(qn.lbfgs_direction(g, run.history), st)
    cfg = qn.StepConfig(min_ascent=run.step_cfg.min_ascent, max_trials=5)
    s0 = st.sweeps
    host = qn.find_step_size(st, d, run.gamma, cfg, on_device=False)
    n_host = st.sweeps - s0
    s0 = st.sweeps
    assert qn.find_step_size(st, d, run.gamma, cfg) == host
    assert st.sweeps - s0 == n_host
    bounds = [r.dual_objective for r in run.records]
    assert all(b1 >= b0 - 1e-9 * max(1.0, abs(b0)) for b0, b1 in zip(bounds, bounds[1:]))
    assert _feasibility(st) < 1e-9
