"""Primal-dual gap of the C3/C4 pairs: solve the dual to its stopping rule,
then recover_primal (agreement fixing + conditioning + exact residual
search) and report the relative primal-dual gap (GPU tool).

usage: python tools/primal_gap.py [config ...]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200 import primal  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.product_space import synthetic_product_space, verify_solution  # noqa: E402
from paper_2310_08230_b200.qn import solve  # noqa: E402

for cfg_name in sys.argv[1:] or ["c3", "c4"]:
    inst = build_instance(cfg_name, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = solve(inst, SolveConfig(mode="hybrid", max_iterations=400), device="cuda:0")
    t1 = time.perf_counter()
    sol = primal.recover_primal(inst, res.state, SolveConfig(max_seconds=60.0))
    t2 = time.perf_counter()
    out = {"config": cfg_name, "dual_iterations": res.iterations, "dual_s": t1 - t0, "best_bound": res.best_bound,
           "primal_s": t2 - t1, "status": sol.status, "ladder_stage": sol.ladder_stage}
    if sol.assignment is not None:
        x = np.asarray(sol.assignment)
        out["primal_objective"] = float(inst.costs @ x)
        out["gap"] = sol.report.primal_dual_gap
        ps = synthetic_product_space(cfg_name, 0)
        out["violated_rows"] = len(verify_solution(ps, x[: ps.num_variables]))
        # gap reached during the dual solve: first iteration within 1e-3 of the primal
        p = out["primal_objective"]
        hit = next((r for r in res.records if (p - r.dual_objective) <= 1e-3 * abs(p)), None)
        out["time_to_1e-3_primal_dual_gap_s"] = hit.time_s if hit else None
        out["iterations_to_1e-3_primal_dual_gap"] = hit.iteration if hit else None
    print(json.dumps(out), flush=True)
