"""Per-phase wall time of C2 solver steps, synchronised between phases (GPU tool).

Mirrors DualSolver.step (paper_2310_08230_b200/qn.py) phase by phase.
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200 import qn  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.dual import BACKWARD, FORWARD, dual_objective, mma_pass, subgradient_device  # noqa: E402
from paper_2310_08230_b200.kernels import dev_sub  # noqa: E402

inst = build_instance("c2", 0)
run = qn.DualSolver(inst, SolveConfig(max_iterations=10**9, dual_tolerance=0.0), device="cuda:0").start()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12


def phase(log, name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    log[name] = round((time.perf_counter() - t) * 1e3, 3)
    return out


for it in range(steps):
    st, h, cfg = run.state, run.history, run.step_cfg
    log = {"it": it + 1, "hist": len(h)}
    t0 = time.perf_counter()
    if len(h) > 0:
        g = phase(log, "subgradient", lambda: subgradient_device(st))
        dh = phase(log, "lbfgs", lambda: qn.lbfgs_direction(g, h))
        d = phase(log, "project", lambda: qn.project_direction(dh, st))
        gamma, better = phase(log, "step_search", lambda: qn.find_step_size(st, d, run.gamma, cfg))
        run.gamma = gamma
        if better:
            phase(log, "shift", lambda: st.shift_lambda_scaled(gamma, d))
    phase(log, "mma_fw", lambda: mma_pass(st, FORWARD))
    phase(log, "mma_bw", lambda: mma_pass(st, BACKWARD))
    bound = phase(log, "objective", lambda: dual_objective(st))
    g_now = phase(log, "subgradient2", lambda: subgradient_device(st))

    def hist():
        s, y = h.reserve(st.lam_d)
        dev_sub(s, st.lam_d, run.lam_prev)
        dev_sub(y, run.g_prev, g_now)
        qn.update_history(s, y, h, cfg)
        run.lam_prev.copy_(st.lam_d)

    phase(log, "history", hist)
    run.g_prev = g_now
    if it == 0:
        cfg.min_ascent = run.cfg.ascent_rel_threshold * (bound - run.initial_bound)
    log["total"] = round((time.perf_counter() - t0) * 1e3, 3)
    log["mem_gb"] = round(torch.cuda.memory_allocated() / 1e9, 2)
    print(json.dumps(log), flush=True)
