"""Phase timing of the merged C5 batch solve (GPU tool): merge, upload +
plans (init_duals), averaging iterations, per-instance bounds; 6 repetitions."""
import gc
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import C5_ITERATIONS, SolveConfigC5, c5_instances  # noqa: E402
from paper_2310_08230_b200.batch import instance_bounds, merge_instances  # noqa: E402
from paper_2310_08230_b200.dual import init_duals  # noqa: E402
from paper_2310_08230_b200.qn import solve  # noqa: E402

insts = c5_instances(range(64))
dev = torch.device("cuda", 0)
for schedule in ("exact", "deferred"):
    cfg = SolveConfigC5(schedule)
    for rep in range(6):
        gc.collect()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m, idx = merge_instances(insts, reuse_buffers=True)
        t1 = time.perf_counter()
        st = init_duals(m, device=dev, schedule=schedule)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res = solve(m, cfg, device=dev, state=st)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        b = instance_bounds(res.state, idx, insts)
        t4 = time.perf_counter()
        print(json.dumps({"schedule": schedule, "rep": rep, "merge": round(t1 - t0, 4), "init": round(t2 - t1, 4),
                          "solve": round(t3 - t2, 4), "bounds": round(t4 - t3, 4), "total": round(t4 - t0, 4),
                          "iters": res.iterations}), flush=True)
        del st, res, m
