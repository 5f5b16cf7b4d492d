import sys, time, json
sys.path.insert(0, ".")
import torch
from bench import build_instance
from paper_2310_08230_b200.config import SolveConfig
from paper_2310_08230_b200.qn import DualSolver, solve
inst = build_instance("c2", 0)
dev = torch.device("cuda", 0)
run = DualSolver(inst, SolveConfig(mode="hybrid", max_iterations=10**9, dual_tolerance=0.0), device=dev).start()
for _ in range(20): run.step()
torch.cuda.synchronize()
for rep in range(3):
    t = time.perf_counter()
    res = solve(inst, SolveConfig(mode="hybrid", max_iterations=150), device=dev, state=run.state)
    ts = [r.time_s for r in res.records]
    d = [round((b - a) * 1e3, 1) for a, b in zip([0.0] + ts[:-1], ts)]
    print(json.dumps({"rep": rep, "total": time.perf_counter() - t, "iters": res.iterations, "first_ms": d[:12], "t48": ts[min(47, len(ts)-1)], "max_ms": max(d)}), flush=True)
