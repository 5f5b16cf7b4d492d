"""GPU timeline of solver iterations (CUPTI via torch.profiler): kernel busy
time vs wall time and the largest idle gaps (GPU tool)."""
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from bench import build_instance  # noqa: E402
from paper_2310_08230_b200.config import SolveConfig  # noqa: E402
from paper_2310_08230_b200.qn import DualSolver  # noqa: E402

inst = build_instance("c2", 0)
run = DualSolver(inst, SolveConfig(max_iterations=10**9, dual_tolerance=0.0), device="cuda:0").start()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):  # past the early iterations
    run.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        run.step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
spans = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
t0, t1 = spans[0][0], max(s[1] for s in spans)
busy = 0
cur_s, cur_e = spans[0][0], spans[0][1]
gaps = []
for s, e, n in spans[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, n))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
agg = {}
for s, e, n in spans:
    k = n.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
    agg[k] = agg.get(k, 0) + (e - s)
print(json.dumps({"wall_us": t1 - t0, "busy_us": busy, "idle_us": (t1 - t0) - busy, "kernels": len(spans),
                  "gaps_over_10us": sum(1 for g in gaps if g[0] > 10), "idle_in_gaps_over_10us": sum(g[0] for g in gaps if g[0] > 10),
                  "top_gaps": sorted(gaps, reverse=True)[:12],
                  "by_kernel_us": dict(sorted(agg.items(), key=lambda kv: -kv[1])[:15])}, indent=1))
