"""Averaging-only (mode mma-only) time to the 1e-3 gap at C4 for both schedules
(GPU tool): how far plain averaging gets without the quasi-Newton step."""
import sys, time, json
sys.path.insert(0, ".")
from bench import build_instance
from paper_2310_08230_b200 import qn
from paper_2310_08230_b200.config import SolveConfig
inst = build_instance("c4", 0)
dstar = 381.2446921751127
for sched in ("deferred", "exact"):
    t = time.perf_counter()
    res = qn.solve(inst, SolveConfig(mode="mma-only", mma_schedule=sched, max_iterations=600, dual_tolerance=-float("inf")), device="cuda:0")
    el = time.perf_counter() - t
    hit = next((r for r in res.records if (dstar - r.dual_objective) / abs(dstar) <= 1e-3), None)
    print(json.dumps({"sched": sched, "iters": res.iterations, "s": el, "hit_it": hit.iteration if hit else None, "hit_t": hit.time_s if hit else None, "final_gap": (dstar - res.best_bound) / dstar}))
