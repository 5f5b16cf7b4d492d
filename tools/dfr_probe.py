"""Deferred vs exact schedule on one GPU: per-iteration cost, per-kernel
CUDA-event times and time to a 1e-3 / 1e-4 relative gap (vs the better of the
two runs' best bounds).  python tools/dfr_probe.py c4 [omega ...]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.dual import KernelTimer, init_duals  # noqa: E402
from paper_2310_08230_b200.qn import DualSolver, solve  # noqa: E402

cfg = sys.argv[1]
omegas = [float(x) for x in sys.argv[2:]] or [0.5]
inst = build_instance(cfg, 0)
dev = torch.device("cuda", 0)
out = {"config": cfg}
runs = {}
for sched, om in [("exact", 0.5)] + [("deferred", w) for w in omegas]:
    st = init_duals(inst, device=dev, schedule=sched)
    torch.cuda.synchronize()
    res = solve(inst, SolveConfig(mode="hybrid", max_iterations=3000 if sched == "deferred" else 600,
                                  mma_schedule=sched, mma_damping=om), device=dev, state=st)
    torch.cuda.synchronize()
    runs[(sched, om)] = res
    # per-kernel timing over 10 steady iterations
    run = DualSolver(inst, SolveConfig(mode="hybrid", max_iterations=10**9, dual_tolerance=0.0, mma_schedule=sched,
                                       mma_damping=om), device=dev, state=st).start()
    for _ in range(5):
        run.step()
    timer = KernelTimer()
    st.pass_timer = timer
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        run.step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    st.pass_timer = None
    out[f"{sched}_{om}"] = {"iterations": res.iterations, "stop": res.stop_reason, "best": res.best_bound,
                           "total_s": res.records[-1].time_s, "ms_per_iteration": dt * 1e3,
                           "kernels": timer.summary()}
best = max(r.best_bound for r in runs.values())
for (sched, om), res in runs.items():
    for gap in (1e-2, 1e-3, 1e-4, 1e-5):
        hit = next((r for r in res.records if best - r.dual_objective <= gap * abs(best)), None)
        out[f"{sched}_{om}"][f"ttg_{gap:g}"] = (hit.time_s, hit.iteration) if hit else None
out["best"] = best
print(json.dumps(out, indent=1))
